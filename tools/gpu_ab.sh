# A/B of variant builds (build_ab/*.so) on the factor + second op, then the step probe.
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
for v in ${AB_VARIANTS:-build_ab/*.so}; do TSQR_LIBRARY=$PWD/$v timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c4 c2}; done > gpurun_out/r2_ab.txt 2>&1
if [ -n "$AB_PROBE" ]; then
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/step_probe 2>/dev/null && /tmp/step_probe > gpurun_out/r2_step_probe.txt 2>&1
nvcc -DTSQR_PROBE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/step_probe2 2>/dev/null && /tmp/step_probe2 > gpurun_out/r2_step_probe_ev.txt 2>&1
fi
cat gpurun_out/r2_ab.txt
