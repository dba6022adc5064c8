# L2 promotion of the TMA copies: DRAM bytes per launch and interleaved A/B of builds
mkdir -p gpurun_out
V="python scripts/ncu_variants.py 512 512 64 zc=0"
for b in "" p0 p1 p2 t0; do
  LB_VARIANT=$b $V > gpurun_out/ncuv_plain.log 2>&1 && LB_VARIANT=$b ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_step --clock-control none -s 2 --csv --log-file gpurun_out/ncu_promo_${b:-def}.csv $V > /dev/null 2>&1
  python - <<PY
import csv
r=[x for x in csv.reader(open('gpurun_out/ncu_promo_${b:-def}.csv')) if len(x)>5]
h=r[0]; i=h.index('Metric Name'); v=h.index('Metric Value')
print('${b:-def}', {row[i]: round(float(row[v].replace(',',''))/(512*512*64),1) if 'bytes' in row[i] else row[v] for row in r[1:]})
PY
done
bash scripts/ab_builds.sh "" p0 3 > gpurun_out/ab_promo.txt 2>&1
bash scripts/ab_builds.sh p1 p2 3 >> gpurun_out/ab_promo.txt 2>&1
cat gpurun_out/ab_promo.txt
