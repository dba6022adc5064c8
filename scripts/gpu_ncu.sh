# ncu full capture of the step kernel: plain run first, then ncu on the same command
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-c3} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for v in ${VARIANTS:-default}; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  if [ "$v" != "default" ]; then LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > /dev/null 2>&1; fi
  $CMD > gpurun_out/plain_$tag.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1; echo ncu_$tag=$?
done
