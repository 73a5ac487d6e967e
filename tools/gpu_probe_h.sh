NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/sp 2>/dev/null && PROBE_ONLY=h timeout 120 /tmp/sp
