# full ncu of the top kernels, summarised on the box (reports too large to bring back)
mkdir -p /tmp/rep
prof() {  # name kernel-regex prof_one-args...
  local name=$1 k=$2; shift 2
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/rep/$name python tools/prof_one.py "$@" > gpurun_out/rn_$name.log 2>&1
  python tools/ncu_raw.py /tmp/rep/$name.ncu-rep > gpurun_out/rn_${name}_raw.txt 2>&1
  python tools/ncu_groups.py /tmp/rep/$name.ncu-rep > gpurun_out/rn_${name}_groups.txt 2>&1
  python tools/ncu_lines.py /tmp/rep/$name.ncu-rep 40 > gpurun_out/rn_${name}_lines.txt 2>&1
}
prof chain_c4 k_chain_factor c4 factor 1
prof csapply_c4 k_cs_apply c4 form_q 1
prof chain_c2 k_chain_factor c2 factor 1
prof wide_c3 k_wide_leaves c3 factor 1
prof chain_c5 k_chain_factor c5 factor 1
prof csapply_c5 k_cs_apply c5 apply_qt 1
cp /tmp/rep/chain_c2.ncu-rep gpurun_out/rn_chain_c2.ncu-rep
du -sh gpurun_out
