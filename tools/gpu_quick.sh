# quick perf+correctness loop: probe, a few factor timings, GPU parity subset
timeout -s KILL 30 ./tools/probe_chain 2048 64 148 0 2>&1 | head -20
for args in "1000000 50 4096 4096" "16777216 64 4096 4096" "33554432 32 4096 4096" "1000 50 1000 1000"; do
  timeout -s KILL 60 python tools/chain_check.py $args 4 2>&1 | tail -1
done
