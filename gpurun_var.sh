#!/bin/bash
# A/B the library variants in build/var on the 10M bench (dev helper); FP64 line + FP32 twin
for rep in 1 ${REPS:+2}; do
for v in build/var/*.so; do
  n=$(basename $v .so)
  CKMPM_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/bench_$n.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); sp=d.get('single_precision',{})
print('$n', '%.4e'%d['value'], {k:round(v,3) for k,v in d['phase_ms'].items()}, 'f32 %.4e'%sp.get('value',0), {k:round(v,3) for k,v in sp.get('phase_ms',{}).items()})" || tail -3 gpurun_out/bench_$n.log
done
done
