for v in base c40n64; do
  echo "== $v"
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "64 or 57 or 63" 2>&1 | tail -1
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 16777216 64 4096 4096 3 | tail -1 | cut -c1-100
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 1000000 60 4096 1024 4 | tail -1 | cut -c1-100
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 200 python tools/kprof.py 16777216 64 4096 4096 64 2 2>&1 | grep cs_apply
done
