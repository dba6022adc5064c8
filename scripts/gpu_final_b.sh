# round-end evidence, part B: ncu launch lists and one --set full capture per step kernel
# (each ncu run after the same command exited 0 without ncu); usage: gpu_final_b.sh name...
mkdir -p gpurun_out
run_ncu() {  # name, kernel regex, bench args
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $3"
  $CMD > gpurun_out/plain_$1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$1.csv $CMD > gpurun_out/ncu1_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o gpurun_out/prof_kstep_$1 $CMD > gpurun_out/ncu2_$1.log 2>&1; echo ncu_$1=$? $(date +%T)
}
for n in "$@"; do
  case $n in
    c5) run_ncu c5 k_step_ws "" ; cp gpurun_out/launches_c5.csv gpurun_out/launches.csv ;;
    c3) run_ncu c3 k_step_ws "--config c3" ;;
    c2) run_ncu c2 k_step_ws "--config c2" ;;
    c4) run_ncu c4 k_step_ws "--config c4" ;;
    mrt) run_ncu mrt k_step_ws "--collision mrt" ;;
    ch) run_ncu ch k_step_ch "--collision ch" ;;
    lc) run_ncu lc k_step_lc "--collision lc" ;;
  esac
done
