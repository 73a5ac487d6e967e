for b in 701 702 699; do CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/tma_diag.py 64 3000 $b 2>&1 | grep -E "^ok|Error" | head -2; done
for b in 701 702; do CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/tma_diag.py 32 3000 $b 2>&1 | grep -E "^ok|Error" | head -2; done
