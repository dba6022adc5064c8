# DRAM bytes per site of the step kernels (tile, probes 1-4, ws) for build variants (';'-separated)
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:- }"
n=0
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > /dev/null 2>&1 || echo build_fail
  timeout 300 python scripts/probe_ncu.py ${CFG:-c5} > /dev/null 2>&1 || echo plain_fail
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step --csv --log-file gpurun_out/bytes_$n.csv python scripts/probe_ncu.py ${CFG:-c5} > /dev/null 2>&1
  echo "[$v]"; python scripts/ncu_bytes.py gpurun_out/bytes_$n.csv ${SITES:-16777216}
  n=$((n+1))
done
