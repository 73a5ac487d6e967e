timeout 900 python -m pytest tests/test_gpu_cholqr.py -q -m gpu > gpurun_out/r2g_tests.txt 2>&1
tail -15 gpurun_out/r2g_tests.txt
