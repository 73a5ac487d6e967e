timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/rr_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rr_ncu_launch.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/rr_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rr_ncu_launch2.log 2>&1
wc -l gpurun_out/rr_launches_c4.csv gpurun_out/rr_launches_c2.csv
