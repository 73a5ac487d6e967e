# time factor variants (A/B): usage bash tools/gpu_ab.sh v1 v2 ...
for v in "$@"; do
  for a in "1000000 50 4096 4096" "16777216 64 4096 4096"; do
    TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 90 python tools/chain_check.py $a 3 2>&1 | tail -1 | sed "s/^/$v: /" | cut -c1-120
  done
done
