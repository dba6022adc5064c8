# where the extra DRAM reads of k_step_ws come from: L2 lookups by eviction class
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
M=dram__sectors_read.sum,dram__sectors_write.sum,lts__d_sectors_fill_device.sum
for p in evict_first evict_last evict_normal; do for h in hit miss; do M=$M,lts__t_sectors_op_read_${p}_lookup_$h.sum,lts__t_sectors_op_write_${p}_lookup_$h.sum; done; done
M=$M,lts__t_sectors_lookup_miss_data_promoted.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum
V="python scripts/ncu_variants.py 512 512 64 zs=0"
$V > gpurun_out/ncuv_plain.log 2>&1 && ncu --metrics $M -k regex:k_step --clock-control none -s 2 --csv --log-file gpurun_out/ncu_l2class.csv $V > gpurun_out/ncu_l2class.log 2>&1; echo ncu=$?
