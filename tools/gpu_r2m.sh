timeout 900 python -m pytest tests/test_gpu_host.py -x -q -m gpu > gpurun_out/r2m_tests.txt 2>&1
tail -15 gpurun_out/r2m_tests.txt
timeout -s KILL 600 python bench.py > gpurun_out/r2m_bench_c4.json 2> gpurun_out/r2m_bench_c4.err
timeout -s KILL 600 python bench.py --config c2 > gpurun_out/r2m_bench_c2.json 2> gpurun_out/r2m_bench_c2.err
python -c "
import json
for c in ('c4','c2'):
    d=json.load(open('gpurun_out/r2m_bench_%s.json'%c)); print(c, d['value'], d['ms_factor'], d['roofline']['frac'], d['second_op_ms'], d['e2e'])
"
