# third-order dlarfg scalars as the default: GPU suite, smoke, C3 A/B vs the Newton-2 build, C4 bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h3_smoke.txt 2>&1; tail -1 gpurun_out/h3_smoke.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/h3_tests.txt 2>&1; tail -2 gpurun_out/h3_tests.txt
{ for r in 1 2 3; do TSQR_LIBRARY=$PWD/ab_tmp/base.so timeout 300 python tools/ab_factor.py c3 c1; TSQR_LIBRARY=$PWD/paper_0808_2664_b200/libtsqr.so timeout 300 python tools/ab_factor.py c3 c1; done; } > gpurun_out/h3_ab.txt 2>&1; cat gpurun_out/h3_ab.txt
timeout -s KILL 900 python bench.py > gpurun_out/h3_bench_c4.json 2> gpurun_out/h3_bench_c4.err; tail -c 200 gpurun_out/h3_bench_c4.json
