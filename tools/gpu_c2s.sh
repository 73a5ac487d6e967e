# C2 tile split s = 1366 (3 tiles per 4096-row block, 735 tiles = 4.97 waves of 148 CTAs) vs 1024
{ for r in 1 2 3; do for s in 1024 1366; do AB_S=$s timeout 300 python tools/ab_factor.py c2; done; done; } > gpurun_out/c2s_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k c2 > gpurun_out/c2s_tests.txt 2>&1
timeout -s KILL 900 python bench.py --config c2 > gpurun_out/c2s_bench_c2.json 2> gpurun_out/c2s_bench_c2.err
cat gpurun_out/c2s_ab.txt; tail -2 gpurun_out/c2s_tests.txt; tail -c 600 gpurun_out/c2s_bench_c2.json
