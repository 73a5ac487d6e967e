set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for s in 64 96 128 192; do timeout 120 python tools/prof_one.py c2 form_q 3 1000000 $s 2>&1 | tail -2; done
timeout 120 python tools/prof_one.py c4 form_q 2 2>&1 | tail -2
timeout 120 python tools/prof_one.py c5 apply_qt 2 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_one.py c2 form_q 1 > gpurun_out/launch_c2.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_factor -c 1 -o gpurun_out/factor_c2 python tools/prof_one.py c2 form_q 1 > gpurun_out/ncu_full.log 2>&1
