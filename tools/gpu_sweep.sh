# tile-size sweep of the factor (chain_check prints R error + device time)
for s in 4096 2048 1366 1024 820 683; do timeout -s KILL 60 python tools/chain_check.py 1000000 50 4096 $s 5 2>&1 | tail -1; done
for s in 4096 2048 1366; do timeout -s KILL 120 python tools/chain_check.py 16777216 64 4096 $s 3 2>&1 | tail -1; done
for s in 4096 2048 1366; do timeout -s KILL 120 python tools/chain_check.py 33554432 32 4096 $s 3 2>&1 | tail -1; done
