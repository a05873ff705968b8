#!/bin/bash
# dev helper: per-launch device times of the bench command (ncu launch list)
cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-chains 1 --no-single ${BENCH_ARGS}"
$cmd > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-400} --csv --log-file gpurun_out/${OUT:-launches}.csv $cmd > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
