# A/B variants of libtsqr.so (developer tool): build/variants/<name>.so
set -e
cd "$(dirname "$0")/../paper_0808_2664_b200"
mkdir -p build/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -shared"
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  ( nvcc $F $defs -o build/variants/$name.so csrc/tsqr_api.cu csrc/tsqr_wy.cu csrc/tsqr_chain.cu csrc/tsqr_cs.cu csrc/tsqr_wide.cu csrc/tsqr_tree.cu csrc/tsqr_caqr.cu csrc/tsqr_stream.cu csrc/tsqr_combine.cu csrc/plan.cpp -lcudart && echo built $name ) &
done
wait
