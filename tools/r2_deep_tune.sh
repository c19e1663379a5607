# c2 / c2' ring depth and L2 prefetch distance sweep (env only)
set -x
for S in 4 5 6 7; do for PF in 0 2 6; do
  OCTGPU_DEEP_S=$S OCTGPU_PREFETCH=$PF P=1.0 K=198 TAG="S=$S pf=$PF" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done; done
for S in 3 4 5; do for PF in 0 4; do
  OCTGPU_DEEP_S=$S OCTGPU_PREFETCH=$PF P=0.5 K=200 TAG="S=$S pf=$PF" timeout 300 python tools/step_timer.py 2>&1 | tail -1
done; done
