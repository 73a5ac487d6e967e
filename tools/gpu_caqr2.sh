export PYTHONPATH=$PWD
for args in "1000000 512 64 4096 1024" "1000000 256 64 4096 1024" "1000000 1024 64 4096 1024" "100000 512 64 4096 1024"; do
  timeout 300 python tools/caqr_time.py $args
done > gpurun_out/r2_caqr.txt 2>&1
cat gpurun_out/r2_caqr.txt
