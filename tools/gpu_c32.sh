# 16 < n <= 32 chunk-configuration variants (developer tool)
for v in base v48x12 v40x12 v32x16 v48x8; do
  echo "== $v"
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "24 or 32" 2>&1 | tail -1
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 33554432 32 4096 4096 3 | tail -1 | cut -c1-110
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 120 python tools/chain_check.py 1000000 24 4096 1024 4 | tail -1 | cut -c1-110
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 200 python tools/kprof.py 33554432 32 4096 4096 128 2 2>&1 | grep cs_apply | cut -c1-60
done
