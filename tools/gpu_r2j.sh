AB_S=1366 python tools/ab_factor.py c2 > gpurun_out/r2j_ab.txt 2>&1
AB_S=1024 python tools/ab_factor.py c2 >> gpurun_out/r2j_ab.txt 2>&1
AB_S=1366 python tools/ab_factor.py c2 >> gpurun_out/r2j_ab.txt 2>&1
python tools/ab_factor.py c3 >> gpurun_out/r2j_ab.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2j_tests.txt 2>&1
cat gpurun_out/r2j_ab.txt; tail -3 gpurun_out/r2j_tests.txt
