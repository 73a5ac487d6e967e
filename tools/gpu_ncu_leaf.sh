# full-ncu captures of the leaf kernel (C4, C2) on the current code (prefix r2g_)
rm -rf /tmp/rep; mkdir -p /tmp/rep
prof() {
  local name=$1 k=$2; shift 2
  timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/rep/$name python tools/prof_one.py "$@" > gpurun_out/r2g_$name.log 2>&1
  python tools/ncu_raw.py /tmp/rep/$name.ncu-rep > gpurun_out/r2g_${name}_raw.txt 2>&1
  python tools/ncu_groups.py /tmp/rep/$name.ncu-rep > gpurun_out/r2g_${name}_groups.txt 2>&1
  python tools/ncu_lines.py /tmp/rep/$name.ncu-rep 40 > gpurun_out/r2g_${name}_lines.txt 2>&1
}
prof chain_c4 k_chain_factor c4 factor 1
prof chain_c2 k_chain_factor c2 factor 1
head -4 gpurun_out/r2g_chain_c4_raw.txt gpurun_out/r2g_chain_c2_raw.txt
