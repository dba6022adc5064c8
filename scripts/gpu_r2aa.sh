# wrapped halo boxes: TMA box + side pieces: parity, schedule trace, A/B against the previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mrt.py tests/test_gpu_ranks.py -q -m gpu -x > gpurun_out/t_side.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_side.log
LB_VARIANT=trace timeout 300 python scripts/trace_schedule.py 512 512 64 "zc=0" > gpurun_out/trace_side_c5.json 2>&1; echo trace=$?
LB_VARIANT=trace timeout 300 python scripts/trace_schedule.py 256 256 256 "zc=0" > gpurun_out/trace_side_c4.json 2>&1; echo trace=$?
cat gpurun_out/trace_side_c5.json gpurun_out/trace_side_c4.json | python -c "
import json,sys
txt=sys.stdin.read().replace('}\n{','}\n@@{')
for part in txt.split('@@'):
    d=json.loads(part)
    for k,v in d.items(): print(k, {x: v[x] for x in ('kernel_us','busy_fraction','sm_end_us_min_p50_max','dur_us_interior_edge')})
"
bash scripts/ab_builds.sh old "" 3 > gpurun_out/ab_side_c5.txt 2>&1
bash scripts/ab_builds.sh old "" 3 --config c4 --steps 100 > gpurun_out/ab_side_c4.txt 2>&1
bash scripts/ab_builds.sh old "" 2 --config c5alt --steps 100 > gpurun_out/ab_side_c5alt.txt 2>&1
cat gpurun_out/ab_side_*.txt
