# ncu launch lists + full captures of the step kernel for the other bench lines (c2, c4, mrt, ch)
mkdir -p gpurun_out
run() {  # name, bench args
  local n=$1; shift
  local CMD="python bench.py $* --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$n.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_$n.csv $CMD > gpurun_out/ncu1_$n.log 2>&1; echo ncu_launches_$n=$?
  ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_kstep_$n $CMD > gpurun_out/ncu2_$n.log 2>&1; echo ncu_full_$n=$?
}
run c2 --config c2
run c4 --config c4
run mrt --collision mrt
run ch --collision ch
