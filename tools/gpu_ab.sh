# A/B of variant builds (build_ab/*.so) on the factor + second op; optional step probe
# variants (PROBE_VARIANTS="name:flags;name2:flags2").
NCCL=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")
for v in ${AB_VARIANTS:-build_ab/*.so}; do TSQR_LIBRARY=$PWD/$v timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c4 c2}; done > gpurun_out/r2_ab.txt 2>&1
if [ -n "$PROBE_VARIANTS" ]; then
  : > gpurun_out/r2_step_probe.txt
  IFS=';' read -ra PV <<< "$PROBE_VARIANTS"
  for pv in "${PV[@]}"; do
    name=${pv%%:*}; flags=${pv#*:}
    nvcc $flags -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_0808_2664_b200/csrc -I $NCCL/include tools/step_probe.cu -o /tmp/sp_$name 2>/dev/null && { echo "== probe $name ($flags)"; /tmp/sp_$name; } >> gpurun_out/r2_step_probe.txt 2>&1
  done
fi
cat gpurun_out/r2_ab.txt
