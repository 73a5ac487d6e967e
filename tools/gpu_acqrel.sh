# A/B on the final code: conforming release/acquire hand-offs (-DTSQR_HANDOFF_ACQREL) and the
# third-order dlarfg scalars (-DTSQR_HOUSE3) against the default build
{ for r in 1 2 3; do for v in base acqrel house3; do TSQR_LIBRARY=$PWD/ab_tmp/$v.so timeout 300 python tools/ab_factor.py c4 c2 c5; done; done; } > gpurun_out/acqrel_ab.txt 2>&1
cat gpurun_out/acqrel_ab.txt
