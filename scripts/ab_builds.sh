# A/B of two builds of the library in alternating processes (same box):
#   bash scripts/ab_builds.sh <variant-a> <variant-b> <rounds> <bench args...>
# variant "" = liblb.so, else liblb_<variant>.so; prints one bench value per run
A=$1; B=$2; N=$3; shift 3
for r in $(seq 1 $N); do
  for v in "$A" "$B"; do
    val=$(LB_VARIANT=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline "$@" 2>gpurun_out/abb_${v:-default}_$r.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
    echo "variant=${v:-default} round=$r $val"
  done
done
