# full GPU suite + bench lines (C4, C2, C5) on the current code
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r3g_tests.txt 2>&1; tail -2 gpurun_out/r3g_tests.txt
for c in c4 c2 c5; do
  timeout -s KILL 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r3g_bench_$c.json 2> gpurun_out/r3g_bench_$c.err
done
python - <<'P'
import json
for c in ("c4","c2","c5"):
    try:
        d=json.load(open(f"gpurun_out/r3g_bench_{c}.json"))
        print(c, "factor", round(d["ms_factor"],4), "leaf", round(d["roofline"]["kernel_ms"],4), "tree", round(d["roofline"]["tree_ms"],4), "frac", round(d["roofline"]["frac"],4), "2nd", round(d["second_op_ms"],4), "e2e ms", round(d["e2e"]["ms_per_step"],2))
    except Exception as e: print(c, "ERR", e)
P
