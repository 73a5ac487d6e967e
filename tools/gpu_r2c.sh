timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/r2i_chain_c4 python tools/prof_one.py c4 factor 1 2097152 > gpurun_out/r2i_ncu.log 2>&1
tail -2 gpurun_out/r2i_ncu.log
