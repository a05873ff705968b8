#!/bin/bash
# quick perf probe used during development: gpu tests (-x) + one bench line + optional ncu of small case
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|^E |FAILED" gpurun_out/pytest_gpu.log | head -10
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('%.3e'%d['value'], {k:round(v,3) for k,v in d['phase_ms'].items()}, d['clocks'])" || tail -5 gpurun_out/bench.log
if [ -n "$NCU" ]; then
  cmd="python bench.py --cells 64 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS}"
  $cmd > gpurun_out/plain_small.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 2 -c 2 -o gpurun_out/$NCUOUT $cmd > gpurun_out/ncu.log 2>&1; echo ncu=$?
fi
