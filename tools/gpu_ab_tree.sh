# A/B of variant libraries (build_ab/*.so) on the given configs + the variant's wide-engine parity tests
V=${V:-wt1}
for r in 1 2; do for v in base $V; do TSQR_LIBRARY=$PWD/build_ab/$v.so timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c3}; done; done > gpurun_out/ab_tree.txt 2>&1
cat gpurun_out/ab_tree.txt
TSQR_LIBRARY=$PWD/build_ab/$V.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -m gpu -x -k "${AB_TESTS:-200 or wide or c3 or 96 or 128}" > gpurun_out/ab_tree_tests.txt 2>&1; tail -3 gpurun_out/ab_tree_tests.txt
