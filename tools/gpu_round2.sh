# round-2 artifacts: edge tests, bench lines (all configs), reference arm, launch list
set -x
timeout 900 python -m pytest tests/test_gpu_edge.py -q -m gpu -x > gpurun_out/rr_edge.txt 2>&1; tail -2 gpurun_out/rr_edge.txt
for c in c4 c2 c3 c5 c1; do
  timeout -s KILL 900 python bench.py --config $c > gpurun_out/rr_bench_$c.json 2> gpurun_out/rr_bench_$c.err
  tail -c 200 gpurun_out/rr_bench_$c.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rr_bench_ref_c4.json 2> gpurun_out/rr_bench_ref_c4.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rr_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rr_ncu_launch.log 2>&1
du -sh gpurun_out
