# A/B of the top-down panel-level node hand-offs (TSQR_NODE_PPIPE_TD) in build_ab/td.so
for r in 1 2; do for e in 0 1; do echo "TD=$e"; TSQR_NODE_PPIPE_TD=$e TSQR_LIBRARY=$PWD/build_ab/td.so timeout 300 python tools/ab_factor.py c2 c4; done; done > gpurun_out/ab_td.txt 2>&1
cat gpurun_out/ab_td.txt
TSQR_NODE_PPIPE_TD=1 TSQR_LIBRARY=$PWD/build_ab/td.so timeout 900 python -m pytest tests -q -m gpu -x -k "form_q or apply_q or formq or c2 or c4 or host or ctx or multirank or caqr or stream or smoke or edge" > gpurun_out/td_tests.txt 2>&1; tail -2 gpurun_out/td_tests.txt
