for r in 1 2; do for v in build_ab/*.so; do TSQR_LIBRARY=$PWD/$v timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c4 c2}; done; done > gpurun_out/ab3.txt 2>&1
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
for f in "" "-DTSQR_EARLY_R"; do nvcc $f -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/sp 2>/dev/null && { echo "== probe $f"; timeout 60 /tmp/sp | grep "n64 c40"; } >> gpurun_out/ab3.txt 2>&1; done
cat gpurun_out/ab3.txt
