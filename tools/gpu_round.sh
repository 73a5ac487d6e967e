# round artifacts: bench lines (all configs), reference arm, launch list + full ncu of the dominant kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for c in ${CONFIGS:-c2 c3 c4 c5 c1}; do
  timeout -s KILL 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -c 300 gpurun_out/bench_$c.err
done
[ -n "$NO_REF" ] || timeout -s KILL 300 python bench.py --impl reference --config c2 --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2>&1
[ -n "$NO_NCU" ] && exit 0
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launch_c2.csv 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/chain_factor_c2 python tools/prof_one.py c2 form_q 1 > gpurun_out/ncu_c2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_wide_leaves -c 1 -o gpurun_out/wide_leaves_c3 python tools/prof_one.py c3 factor 1 > gpurun_out/ncu_c3.log 2>&1
[ -n "$NCU_C4" ] && timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/chain_factor_c4 python tools/prof_one.py c4 factor 1 > gpurun_out/ncu_c4.log 2>&1
[ -n "$CUSOLVER" ] && PYTHONPATH=$PWD timeout -s KILL 300 python tools/caqr_time.py 1000000 50 64 4096 1024 > gpurun_out/cusolver_c2.txt 2>&1
exit 0
