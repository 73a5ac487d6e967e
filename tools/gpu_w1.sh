for v in base w1cta; do
  echo "== $v"
  for s in 400 342 700 1024; do
    TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 100000 200 2048 $s 4 | tail -1 | cut -c1-110
  done
done
TSQR_LIBRARY=paper_0808_2664_b200/build/variants/w1cta.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "200 or 224 or 100" 2>&1 | tail -1
