# ncu DRAM bytes per launch for L2 policy / order / z-chunk variants at 512x512x64
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
V="gt=1 gt=0 gt=3 gt=2 box=0 ft=0 band=2 zc=16 zc=64 gt=0,zc=64 gt=1"
timeout 600 python scripts/ncu_variants.py 512 512 64 $V > gpurun_out/ncuvar_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_step --csv --log-file gpurun_out/ncu_variants.csv python scripts/ncu_variants.py 512 512 64 $V > gpurun_out/ncuvar.log 2>&1; echo ncuvar=$?
timeout 600 python scripts/ab_tune.py 512 512 64 gt=1 gt=0 gt=3 --rounds 4 > gpurun_out/ab_gt.json 2>&1; echo ab=$?; cat gpurun_out/ab_gt.json
