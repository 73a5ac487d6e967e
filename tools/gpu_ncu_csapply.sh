# full ncu of the C4 form-Q leaf kernel (k_cs_apply) on the final code
rm -rf /tmp/rep; mkdir -p /tmp/rep
timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:k_cs_apply -c 1 -o /tmp/rep/csapply_c4 python tools/prof_one.py c4 form_q 1 > gpurun_out/r2k_csapply_c4.log 2>&1
python tools/ncu_raw.py /tmp/rep/csapply_c4.ncu-rep > gpurun_out/r2k_csapply_c4_raw.txt 2>&1
python tools/ncu_groups.py /tmp/rep/csapply_c4.ncu-rep > gpurun_out/r2k_csapply_c4_groups.txt 2>&1
grep -E "gpu__time_duration.sum|dram__bytes_(read|write).sum |sm__pipe_fp64_cycles_active|sm__inst_executed_pipe_dmma|launch__occupancy_limit|sm__warps_active.avg.pct|launch__registers" gpurun_out/r2k_csapply_c4_raw.txt | head -20
