for v in default m16_3 m8_3 m8_2 m4_4; do
  if [ $v = default ]; then unset OCTGPU_LIB; else export OCTGPU_LIB=tools/variants/$v/liboctgpu.so; fi
  echo "== $v"; timeout 300 python tools/measure_timer.py
done
unset OCTGPU_LIB
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "golden or heights or invariant or measure or balances" 2>&1 | tail -2
