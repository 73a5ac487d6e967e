timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_cs_apply -c 1 -o gpurun_out/r2f_csapply_c4 python tools/prof_one.py c4 form_q 1 2097152 > gpurun_out/r2f_ncu.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_cs_apply -c 1 -o gpurun_out/r2f_csapply_c5 python tools/prof_one.py c5 apply_qt 1 2097152 > gpurun_out/r2f_ncu5.log 2>&1
tail -2 gpurun_out/r2f_ncu.log gpurun_out/r2f_ncu5.log
