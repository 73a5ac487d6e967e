for args in "1000000 50 4096 4096" "1000000 50 4096 1366" "16777216 64 4096 4096" "33554432 32 4096 4096" "1000 50 1000 1000" "100000 7 4096 256"; do
  timeout -s KILL 60 python tools/chain_check.py $args 4 2>&1 | tail -2
done
timeout -s KILL 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
