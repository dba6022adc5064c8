# build-variant sweep of scripts/probe.py (variants separated by ';'), REPEAT runs
# each, interleaved, median reported per variant
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
n=0
for v in "${VS[@]}"; do
  mkdir -p gpurun_out/var$n
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo "build_fail [$v]"; tail -5 gpurun_out/build.log; }
  cp paper_1609_01479_b200/liblb.so gpurun_out/var$n/liblb.so
  n=$((n+1))
done
for rep in $(seq 1 ${REPEAT:-1}); do
  n=0
  for v in "${VS[@]}"; do
    cp gpurun_out/var$n/liblb.so paper_1609_01479_b200/liblb.so
    for cfg in ${CFGS:-c5}; do
      python scripts/probe.py --config $cfg ${PROBE_ONLY:+--only $PROBE_ONLY} > gpurun_out/var$n/probe_${cfg}_$rep.json 2>gpurun_out/probe_v.err || { echo "probe_fail [$v]"; tail -3 gpurun_out/probe_v.err; }
    done
    n=$((n+1))
  done
done
n=0
for v in "${VS[@]}"; do
  for cfg in ${CFGS:-c5}; do
    python - "$v" "$cfg" gpurun_out/var$n <<'PY'
import glob, json, statistics, sys
v, cfg, d = sys.argv[1:4]
runs = [json.load(open(f)) for f in sorted(glob.glob(f"{d}/probe_{cfg}_*.json"))]
keys = [k for k, x in runs[0].items() if isinstance(x, dict) and "mlups" in x]
med = {k: round(statistics.median(r[k]["mlups"] for r in runs)) for k in keys}
print(f"[{v}] {cfg} n={len(runs)}", " ".join(f"{k}={x}" for k, x in med.items()),
      "runs:", {k: [round(r[k]["mlups"]) for r in runs] for k in keys})
PY
  done
  n=$((n+1))
done
rm -rf gpurun_out/var*
