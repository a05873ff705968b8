mkdir -p gpurun_out
for v in default build/var_NOB.so; do
  if [ $v = default ]; then unset CKMPM_B200_LIB; else export CKMPM_B200_LIB=$PWD/$v; fi
  timeout 300 python tools/time_phases.py
  PREC=4 timeout 300 python tools/time_phases.py
done
unset CKMPM_B200_LIB
FUSED=0 timeout 300 python tools/time_phases.py
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -3
