#!/bin/bash
# A/B the library variants in build/var on the 10M bench (dev helper)
for v in build/var/*.so; do
  CKMPM_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/bench_$(basename $v .so).log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$(basename $v .so).log').read().strip().splitlines()[-1]); print('$(basename $v)', '%.3e'%d['value'], {k:round(v,3) for k,v in d['phase_ms'].items()})" || tail -3 gpurun_out/bench_$(basename $v .so).log
done
