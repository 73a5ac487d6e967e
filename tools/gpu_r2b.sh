set -x
timeout 600 python bench.py > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo bench rc=$?
timeout 600 python bench.py --config c2 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo bench2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref_c4.json 2> gpurun_out/r2_bench_ref_c4.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1; echo ncu rc=$?
