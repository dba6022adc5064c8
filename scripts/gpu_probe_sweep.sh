# build-variant sweep of scripts/probe.py (variants separated by ';')
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo "build_fail [$v]"; tail -5 gpurun_out/build.log; continue; }
  for cfg in ${CFGS:-c5}; do
    python scripts/probe.py --config $cfg > gpurun_out/probe_v.json 2>gpurun_out/probe_v.err || { echo "probe_fail [$v]"; tail -3 gpurun_out/probe_v.err; continue; }
    python -c "import json;d=json.load(open('gpurun_out/probe_v.json'));print('[$v] $cfg', ' '.join(f\"{k}={round(d[k]['mlups'])}\" for k in ('step','probe1_copy_push','probe2_plus_halo_phi_P','k_stream_site_parallel')), 'copy_gbs', round(d['torch_copy_same_bytes']['gbs']))"
  done
done
