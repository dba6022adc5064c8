# interleaved A/B of two step kernels (probe.py --ab) under several builds of
# liblb.so (abl/liblb_<name>.so):  AB=3,5 CFG=c5 bash scripts/ab_probe_libs.sh name1 name2 ...
mkdir -p gpurun_out
cp paper_1609_01479_b200/liblb.so abl/liblb_keep.so
for v in "$@"; do
  cp abl/liblb_$v.so paper_1609_01479_b200/liblb.so
  for c in ${CFG:-c5}; do
    timeout 300 python scripts/probe.py --config $c --ab ${AB:-3,5} --steps 10 --rounds ${ROUNDS:-10} > gpurun_out/abp_${v}_$c.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/abp_${v}_$c.json'));print('$v', '$c', {k:round(x['mlups']) for k,x in d.items() if k.startswith('ab')})" || tail -3 gpurun_out/abp_${v}_$c.json
  done
done
cp abl/liblb_keep.so paper_1609_01479_b200/liblb.so
