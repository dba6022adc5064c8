mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo b5=$?
python bench.py --config c3 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1; echo b3=$?
python bench.py --config c2 --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2>&1; echo b2=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo bref=$?
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_kstep $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
