python tools/ab_factor.py c4 c2 c5 > gpurun_out/r2n_ab.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2n_tests.txt 2>&1
cat gpurun_out/r2n_ab.txt; tail -2 gpurun_out/r2n_tests.txt
