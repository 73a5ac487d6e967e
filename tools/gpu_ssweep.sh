# tile-split sweep (s = tile rows within b-row blocks) for C2, C4, C5 on the default library
{ for s in 512 768 1024 1366 2048 4096; do AB_S=$s timeout 300 python tools/ab_factor.py c2; done
  for s in 2048 4096; do AB_S=$s timeout 300 python tools/ab_factor.py c4; done
  for s in 2048 4096; do AB_S=$s timeout 300 python tools/ab_factor.py c5; done
  for s in 300 342 400 512 683; do AB_S=$s timeout 300 python tools/ab_factor.py c3; done; } > gpurun_out/ssweep.txt 2>&1
cat gpurun_out/ssweep.txt
