mkdir -p gpurun_out
for v in default build/var_prev.so; do
  if [ $v = default ]; then unset CKMPM_B200_LIB; else export CKMPM_B200_LIB=$PWD/$v; fi
  FUSED=0 MODEL=drucker_prager timeout 300 python tools/time_phases.py
done
unset CKMPM_B200_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_quad.py tests/test_gpu_fused.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_atsize.py -q -x -k "c3 or c4 or twisting or clamp" 2>&1 | tail -3
