#!/bin/bash
# round-end measurement: full bench line (with cpu baseline) + reference arm + launch list
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
OUT=${ROUND_OUT:-launches_round} ./gpurun_launches.sh
