# the Cahn-Hilliard kernel's DRAM bytes per launch (its --set full capture stalls under ncu's
# instrumented replay; the metrics alone replay fine), after the same command exits 0
mkdir -p gpurun_out
CMD="python bench.py --collision ch --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_ch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_step_ch -s 3 -c 1 --csv --log-file gpurun_out/ncu_ch_dram.csv $CMD > gpurun_out/ncu3_ch.log 2>&1; echo ncu_ch=$?
