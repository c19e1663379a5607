set -x
export OCTGPU_DEEP=2 X=1024 Y=320 K=3 KWARM=0 P=1.0
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device python tools/step_timer.py 2>&1 | head -60
OCTGPU_DEEP_L=4 timeout 300 compute-sanitizer --tool memcheck python tools/step_timer.py 2>&1 | head -30
