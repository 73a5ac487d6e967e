# re-check of earlier-neutral variants on the final code: nearest-cut partition, W^T split off / 4 blocks
{ for r in 1 2 3; do for v in base nearest wt0 wt4; do TSQR_LIBRARY=$PWD/ab_tmp/$v.so timeout 300 python tools/ab_factor.py c4 c2 c5; done; done; } > gpurun_out/variants2_ab.txt 2>&1
cat gpurun_out/variants2_ab.txt
