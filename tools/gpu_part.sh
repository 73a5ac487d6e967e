# chain-partition variants (developer tool)
for v in nearest optimal; do
  echo "== $v"
  for s in 1024 1366 683; do
    TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 1000000 50 4096 $s 6 | tail -1 | cut -c1-100
  done
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 16777216 64 4096 4096 3 | tail -1 | cut -c1-100
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 33554432 32 4096 4096 3 | tail -1 | cut -c1-100
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 200 python tools/kprof.py 1000000 50 4096 1024 50 3 2>&1 | grep -E "chain_factor|cs_apply|tree_pipe" | cut -c1-70
done
TSQR_LIBRARY=paper_0808_2664_b200/build/variants/optimal.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
