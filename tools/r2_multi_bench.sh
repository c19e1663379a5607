# N-rank bench on ONE GPU (time-sliced protocol check: OCTGPU_BENCH_ONE_GPU=1)
set -x
export OCTGPU_BENCH_ONE_GPU=1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/r2mb_n$N.json 2> gpurun_out/r2mb_n$N.err; tail -c 1500 gpurun_out/r2mb_n$N.json; tail -3 gpurun_out/r2mb_n$N.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 20 --warmup 3 --config c5 --no-configs --no-cpu-baseline --no-e2e > gpurun_out/r2mb_c5_n$N.json 2> gpurun_out/r2mb_c5_n$N.err; tail -c 800 gpurun_out/r2mb_c5_n$N.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/r2mb_ref_n2.json 2>&1; tail -c 600 gpurun_out/r2mb_ref_n2.json
