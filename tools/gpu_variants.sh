for v in base gw gwgp; do
  echo "== $v"
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "test_factor_r_and_reflectors" 2>&1 | tail -1
  TSQR_LIBRARY=paper_0808_2664_b200/build/variants/$v.so timeout -s KILL 60 python tools/chain_check.py 1000000 50 4096 1024 4 | tail -1 | cut -c1-100
done
