# per-launch time and DRAM bytes of the banded exchange (512x512x64) against one wave (512x64x64)
mkdir -p gpurun_out
export LB_ZCHUNK=64
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed
for lat in 512,512,64 512,64,64; do
  timeout 300 python scripts/run_kernel.py --lattice $lat --kernel 5 --steps 2 > /dev/null 2>&1 || echo plain_fail
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/bandncu_${lat//,/x}.csv python scripts/run_kernel.py --lattice $lat --kernel 5 --steps 2 > /dev/null 2>&1; echo ncu=$?
done
