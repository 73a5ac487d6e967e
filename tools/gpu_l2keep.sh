# A/B: L2 evict_last hint on the wide engine's C row pairs (ab_tmp/{base,keep}.so), C3
for r in 1 2 3; do for v in ab_tmp/base.so ab_tmp/keep.so; do TSQR_LIBRARY=$PWD/$v timeout 300 python tools/ab_factor.py c3; done; done > gpurun_out/l2keep_ab.txt 2>&1
for v in base keep; do TSQR_LIBRARY=$PWD/ab_tmp/$v.so timeout 600 ncu --kernel-name regex:k_wide_leaves --launch-skip 2 -c 2 --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct python tools/ab_factor.py c3 > gpurun_out/l2keep_ncu_$v.txt 2>&1; done
tail -n 30 gpurun_out/l2keep_ab.txt; grep -E "dram__|gpu__time|hit_rate" gpurun_out/l2keep_ncu_*.txt
