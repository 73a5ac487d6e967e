# final round-2 artifacts (prefix r2i_): smoke, full GPU suite, bench lines (all configs), reference
# arm, launch lists (C4, C2), full-ncu summaries of the dominant kernels, N = 2 functional check
# of the bench path (gloo, one GPU)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2i_smoke.txt 2>&1; tail -1 gpurun_out/r2i_smoke.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2i_tests.txt 2>&1; tail -2 gpurun_out/r2i_tests.txt
for c in c4 c2 c3 c5 c1; do
  timeout -s KILL 900 python bench.py --config $c > gpurun_out/r2i_bench_$c.json 2> gpurun_out/r2i_bench_$c.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2i_bench_ref_c4.json 2> gpurun_out/r2i_bench_ref_c4.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/r2i_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_ncu_launch.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv --log-file gpurun_out/r2i_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_ncu_launch2.log 2>&1
rm -rf /tmp/rep; mkdir -p /tmp/rep
prof() {
  local name=$1 k=$2; shift 2
  timeout -s KILL 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/rep/$name python tools/prof_one.py "$@" > gpurun_out/r2i_$name.log 2>&1
  python tools/ncu_raw.py /tmp/rep/$name.ncu-rep > gpurun_out/r2i_${name}_raw.txt 2>&1
  python tools/ncu_groups.py /tmp/rep/$name.ncu-rep > gpurun_out/r2i_${name}_groups.txt 2>&1
  python tools/ncu_lines.py /tmp/rep/$name.ncu-rep 40 > gpurun_out/r2i_${name}_lines.txt 2>&1
}
prof chain_c4 k_chain_factor c4 factor 1
prof chain_c2 k_chain_factor c2 factor 1
prof csapply_c4 k_cs_apply c4 form_q 1
prof wide_c3 k_wide_leaves c3 factor 1
bash tools/gpu_n2.sh > gpurun_out/r2i_n2.txt 2>&1
du -sh gpurun_out
