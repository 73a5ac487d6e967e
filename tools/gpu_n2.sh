# functional check of the N > 1 bench path on one GPU (gloo, both ranks on cuda:0): never a scaling number
export TSQR_BENCH_BACKEND=gloo TSQR_BENCH_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > gpurun_out/n2_c2.json 2> gpurun_out/n2_c2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config c3 --steps 3 --warmup 3 > gpurun_out/n2_c3.json 2> gpurun_out/n2_c3.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --impl reference --gpus 2 --config c2 --steps 3 --warmup 3 > gpurun_out/n2_ref.json 2> gpurun_out/n2_ref.err; echo rc=$?
head -c 400 gpurun_out/n2_c2.json; echo; head -c 300 gpurun_out/n2_c3.json; echo; head -c 200 gpurun_out/n2_ref.json; tail -3 gpurun_out/n2_c2.err
