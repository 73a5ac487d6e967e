# A/B timing of several variant libraries (build_ab/<name>.so) against build_ab/base.so (developer tool)
# usage: VS="v1 v2" AB_CONFIGS="c4 c2" bash tools/gpu_ab_multi.sh
for r in 1 2; do for v in base $VS; do TSQR_LIBRARY=$PWD/build_ab/$v.so timeout 300 python tools/ab_factor.py ${AB_CONFIGS:-c4 c2}; done; done > gpurun_out/ab_multi.txt 2>&1
cat gpurun_out/ab_multi.txt
