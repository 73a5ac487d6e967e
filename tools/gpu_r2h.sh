timeout 900 python -m pytest tests/test_gpu_streamed.py -q -m gpu > gpurun_out/r2h_tests.txt 2>&1
tail -5 gpurun_out/r2h_tests.txt
python tools/stream_q_time.py 4194304 64 1048576 4096 4096 64 > gpurun_out/r2h_streamq.txt 2>&1
python tools/stream_q_time.py 16777216 64 4194304 4096 4096 64 >> gpurun_out/r2h_streamq.txt 2>&1
PYTHONPATH=$PWD python tools/stream_time.py 16777216 64 4194304 4096 4096 >> gpurun_out/r2h_streamq.txt 2>&1
cat gpurun_out/r2h_streamq.txt
