mkdir -p gpurun_out
python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo build_fail; tail gpurun_out/build.log; }
timeout 300 python scripts/ws_diff.py > gpurun_out/ws_diff.log 2>&1; echo ws_diff=$?; cat gpurun_out/ws_diff.log | tail -20
timeout 300 python scripts/probe.py --config c5 --steps 50 > gpurun_out/probe_c5.json 2>gpurun_out/probe_c5.err; echo probe=$?
python -c "import json;d=json.load(open('gpurun_out/probe_c5.json'));print({k:(round(v['mlups']) if isinstance(v,dict) and 'mlups' in v else v) for k,v in d.items()})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:k_step --csv --log-file gpurun_out/probe_ncu.csv python scripts/probe_ncu.py c5 > gpurun_out/probe_ncu.log 2>&1; echo ncu=$?
