# iteration loop on the GPU box: per-kernel times at the main configs, then GPU parity
for a in "1000000 50 4096 4096" "1000000 50 4096 1366" "16777216 64 4096 4096" "33554432 32 4096 4096"; do
  timeout -s KILL 120 python tools/kprof.py $a 2>&1 | grep -v "Warn\|warn"
done
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
