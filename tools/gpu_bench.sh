set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for c in c2 c4 c5 c1; do timeout -s KILL 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.err; done
timeout -s KILL 300 python bench.py --impl reference --config c2 --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_one.py c2 form_q 1 > gpurun_out/launch_c2.csv 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/chain_factor_c2 python tools/prof_one.py c2 form_q 1 > gpurun_out/ncu_c2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/chain_factor_c4 python tools/prof_one.py c4 form_q 1 1048576 > gpurun_out/ncu_c4.log 2>&1
