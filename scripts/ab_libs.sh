# A/B of two builds of liblb.so (ab/liblb_old.so vs ab/liblb_new.so), alternating,
# same process arguments: bench.py lines into gpurun_out/ab_*.json
#   bash scripts/ab_libs.sh "<bench args>" [rounds]
ARGS=${1:-"--steps 100 --no-e2e --no-cpu-baseline"}
R=${2:-3}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for v in old new; do
    cp ab/liblb_$v.so paper_1609_01479_b200/liblb.so
    timeout 300 python bench.py $ARGS > gpurun_out/ab_${v}_$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$i.json'));print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
cp ab/liblb_new.so paper_1609_01479_b200/liblb.so
