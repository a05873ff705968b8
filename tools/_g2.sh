mkdir -p gpurun_out
for v in default build/var_aos.so; do
  if [ $v = default ]; then unset CKMPM_B200_LIB; else export CKMPM_B200_LIB=$PWD/$v; fi
  FUSED=0 timeout 300 python tools/time_phases.py
done
