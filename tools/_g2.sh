for v in default build/var_nopf.so; do
  if [ $v = default ]; then unset CKMPM_B200_LIB; else export CKMPM_B200_LIB=$PWD/$v; fi
  timeout 300 python tools/time_phases.py
  PREC=4 timeout 300 python tools/time_phases.py
  MODEL=drucker_prager timeout 300 python tools/time_phases.py
done
unset CKMPM_B200_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quad.py tests/test_gpu_frame.py tests/test_gpu_dense.py -q -x 2>&1 | tail -3
