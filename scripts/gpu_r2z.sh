# block schedule trace of k_step_ws (measurement build liblb_trace.so)
mkdir -p gpurun_out
LB_VARIANT=trace timeout 300 python scripts/trace_schedule.py 512 512 64 "zc=0" "zc=16" "zc=64" > gpurun_out/trace_c5.json 2>&1; echo trace=$?
LB_VARIANT=trace timeout 300 python scripts/trace_schedule.py 256 256 256 "zc=0" > gpurun_out/trace_c4.json 2>&1; echo trace=$?
python -c "
import json
for f in ['trace_c5','trace_c4']:
    d=json.load(open('gpurun_out/'+f+'.json'))
    for k,v in d.items(): print(f,k,v)
"
