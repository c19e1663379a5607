# Round-2 GPU check: at-scale parity, full GPU suite, default bench line, reference arm.
set -x
nvidia-smi -L; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
timeout 1500 python -m pytest tests/test_scale_gpu.py -x -q -s --durations=10 2>&1 | tail -25
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_scale_gpu.py 2>&1 | tail -6
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -c 4000 gpurun_out/r2a_bench.json; tail -5 gpurun_out/r2a_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; tail -c 1500 gpurun_out/r2a_ref.json
