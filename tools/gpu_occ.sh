# form-Q / apply leaves at 1 vs 2 CTAs per SM (grid = 148 x occ), dev build -DTSQR_APPLY_OCC_ENV
{ for r in 1 2; do for o in 2 1; do for c in c2 c4 c5; do TSQR_APPLY_OCC=$o TSQR_LIBRARY=$PWD/ab_tmp/occenv.so timeout 300 python tools/ab_factor.py $c | sed "s/^/occ=$o /"; done; done; done
  for s in 4096 2048; do for o in 2 1; do TSQR_APPLY_OCC=$o AB_S=$s TSQR_LIBRARY=$PWD/ab_tmp/occenv.so timeout 300 python tools/ab_factor.py c2 | sed "s/^/occ=$o /"; done; done; } > gpurun_out/occ_ab.txt 2>&1
cat gpurun_out/occ_ab.txt
