# ncu source-level stall profile of the step probe (one warp per SM, n = 64, steps only)
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
nvcc ${PROBE_FLAGS} -lineinfo -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/sp || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_probe --launch-skip ${PROBE_SKIP:-1} --launch-count 1 -o gpurun_out/r2_probe /tmp/sp > gpurun_out/r2_ncu_probe.log 2>&1
echo ncu rc=$?
