python tools/ab_factor.py c2 > gpurun_out/r2d_ab.txt 2>&1
AB_S=1024 python tools/ab_factor.py c2 >> gpurun_out/r2d_ab.txt 2>&1
AB_S=2048 python tools/ab_factor.py c2 >> gpurun_out/r2d_ab.txt 2>&1
TSQR_NO_TMA=1 AB_S=1024 python tools/ab_factor.py c2 >> gpurun_out/r2d_ab.txt 2>&1
python tools/ab_factor.py c4 c5 >> gpurun_out/r2d_ab.txt 2>&1
cat gpurun_out/r2d_ab.txt
