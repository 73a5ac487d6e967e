# compact apply slot as the default: GPU suite, smoke, C4 and C5 bench lines
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/sl_smoke.txt 2>&1; tail -1 gpurun_out/sl_smoke.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/sl_tests.txt 2>&1; tail -2 gpurun_out/sl_tests.txt
timeout -s KILL 900 python bench.py > gpurun_out/sl_bench_c4.json 2> gpurun_out/sl_bench_c4.err
timeout -s KILL 900 python bench.py --config c5 > gpurun_out/sl_bench_c5.json 2> gpurun_out/sl_bench_c5.err
timeout -s KILL 900 python bench.py --config c2 > gpurun_out/sl_bench_c2.json 2> gpurun_out/sl_bench_c2.err
ls -la gpurun_out/sl_*
