set -x
free -g; nproc; nvidia-smi -L; cat /proc/cpuinfo | grep "model name" | head -1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_ctx.py -q -m gpu -x -s > gpurun_out/r2_t_edge.log 2>&1; echo edge rc=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -s > gpurun_out/r2_t_full.log 2>&1; echo full rc=$?
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/r2_t_rest.log 2>&1; echo rest rc=$?
timeout 600 python bench.py > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo bench rc=$?
timeout 600 python bench.py --config c2 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo bench2 rc=$?
