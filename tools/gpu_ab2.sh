# A/B of build_ab/*.so variants: C4, C2, C5 factor + second op (two rounds to see noise)
for r in 1 2; do for v in ${AB_VARIANTS:-build_ab/*.so}; do TSQR_LIBRARY=$PWD/$v timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c4 c2 c5}; done; done > gpurun_out/ab2.txt 2>&1
cat gpurun_out/ab2.txt
