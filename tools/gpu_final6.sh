# final round-2 check (prefix r2j_): smoke, full GPU suite, bench lines C4 (default) and C2 (s = 1366),
# the C2 launch list and full-ncu of the C2 leaf kernel at s = 1366, N = 2 functional check
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.txt 2>&1; tail -1 gpurun_out/r2j_smoke.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2j_tests.txt 2>&1; tail -2 gpurun_out/r2j_tests.txt
timeout -s KILL 900 python bench.py > gpurun_out/r2j_bench_c4.json 2> gpurun_out/r2j_bench_c4.err
timeout -s KILL 900 python bench.py --config c2 > gpurun_out/r2j_bench_c2.json 2> gpurun_out/r2j_bench_c2.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/r2j_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_ncu_launch2.log 2>&1
rm -rf /tmp/rep; mkdir -p /tmp/rep
timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o /tmp/rep/chain_c2 python tools/prof_one.py c2 factor 1 > gpurun_out/r2j_chain_c2.log 2>&1
python tools/ncu_raw.py /tmp/rep/chain_c2.ncu-rep > gpurun_out/r2j_chain_c2_raw.txt 2>&1
python tools/ncu_groups.py /tmp/rep/chain_c2.ncu-rep > gpurun_out/r2j_chain_c2_groups.txt 2>&1
python tools/ncu_lines.py /tmp/rep/chain_c2.ncu-rep 40 > gpurun_out/r2j_chain_c2_lines.txt 2>&1
bash tools/gpu_n2.sh > gpurun_out/r2j_n2.txt 2>&1
tail -c 300 gpurun_out/r2j_bench_c4.json; tail -c 300 gpurun_out/r2j_bench_c2.json; grep -E "dram__bytes_(read|write).sum |gpu__time_duration.sum" gpurun_out/r2j_chain_c2_raw.txt | head; cat gpurun_out/r2j_n2.txt | tail -5
