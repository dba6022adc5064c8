mkdir -p gpurun_out
python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo build_fail; tail gpurun_out/build.log; }
for cfg in c5 c3; do
  timeout 300 python scripts/probe.py --config $cfg --ab 1,3 --steps 10 --rounds 20 > gpurun_out/ab_$cfg.json 2>&1; echo ab=$?; cat gpurun_out/ab_$cfg.json
done
timeout 300 python scripts/probe_ncu.py c5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_ws -c 1 -o gpurun_out/prof_ws python scripts/probe_ncu.py c5 > gpurun_out/ncu_ws.log 2>&1; echo ncu=$?
