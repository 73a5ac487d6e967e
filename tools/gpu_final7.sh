# bench lines of every config on the final code (prefix r2k_), reference arm, C4 launch list
for c in c2 c3 c5 c1; do
  timeout -s KILL 900 python bench.py --config $c > gpurun_out/r2k_bench_$c.json 2> gpurun_out/r2k_bench_$c.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_bench_ref_c4.json 2> gpurun_out/r2k_bench_ref_c4.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/r2k_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_ncu_launch.log 2>&1
ls -la gpurun_out/r2k_*
