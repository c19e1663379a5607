set -x
timeout 900 python -m pytest tests/test_p2p_ipc_gpu.py -x -q 2>&1 | tail -2
export OCTGPU_BENCH_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-configs --no-cpu-baseline --no-e2e > gpurun_out/r2g2_n2.json 2> gpurun_out/r2g2_n2.err; tail -c 600 gpurun_out/r2g2_n2.json
