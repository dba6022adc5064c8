# A/B/C... of several builds of liblb.so (abl/liblb_<name>.so, built on the CPU box
# with LB_NVCC_FLAGS), alternating round by round in fresh processes:
#   ARGS="<bench args>" R=<rounds> bash scripts/ab_multi.sh name1 name2 ...
ARGS=${ARGS:-"--steps 100 --no-e2e --no-cpu-baseline"}
R=${R:-3}
mkdir -p gpurun_out
cp paper_1609_01479_b200/liblb.so abl/liblb_keep.so
for i in $(seq 1 $R); do
  for v in "$@"; do
    cp abl/liblb_$v.so paper_1609_01479_b200/liblb.so
    timeout 300 python bench.py $ARGS > gpurun_out/ab_${v}_$i.json 2>gpurun_out/ab_${v}_$i.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$i.json'));print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/ab_${v}_$i.err
  done
done
cp abl/liblb_keep.so paper_1609_01479_b200/liblb.so
