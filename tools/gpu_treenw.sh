# narrow tree: nodes (warps) per block 2 / 4 (default) / 8 on the final code
{ for r in 1 2 3; do for v in base tnw2 tnw8; do TSQR_LIBRARY=$PWD/ab_tmp/$v.so timeout 300 python tools/ab_factor.py c4 c2 c5; done; done; } > gpurun_out/treenw_ab.txt 2>&1
cat gpurun_out/treenw_ab.txt
