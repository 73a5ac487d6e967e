# A/B of library variants (build/variants/*.so): parity subset + C2/C4 factor timing
for v in ${VARIANTS:-base}; do
  echo "== $v"
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "test_factor_r_and_reflectors" 2>&1 | tail -1
  for a in "1000000 50 4096 1024" "16777216 64 4096 4096"; do
    TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 90 python tools/chain_check.py $a 4 | tail -1 | cut -c1-100
  done
done
