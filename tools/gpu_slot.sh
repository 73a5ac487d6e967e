# apply / form-Q slot without the unused row-major region (smem per CTA 93 -> 51 KB at n = 64)
{ for r in 1 2 3; do for v in base compact; do TSQR_LIBRARY=$PWD/ab_tmp/$v.so timeout 300 python tools/ab_factor.py c4 c2 c5; done; done; } > gpurun_out/slot_ab.txt 2>&1
cat gpurun_out/slot_ab.txt
