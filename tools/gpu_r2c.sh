# step probe (1/4/8 warps) + full ncu of the C4-shaped chain kernel (2M rows) with source
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
nvcc -lineinfo -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/sp && timeout 120 /tmp/sp > gpurun_out/r2c_probe.txt 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_factor -c 1 -o gpurun_out/r2c_chain_c4 python tools/prof_one.py c4 factor 1 2097152 > gpurun_out/r2c_ncu.log 2>&1
echo done
