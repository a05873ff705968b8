#!/bin/bash
# dev helper: ncu --set full of the transfer kernels on the 2M-particle case (cells 64)
cmd="python bench.py --cells ${CELLS:-64} --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS}"
$cmd > gpurun_out/plain_small.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:"${NCU:-p2g_tile|g2p_tile}" -s ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/${NCUOUT:-prof} $cmd > gpurun_out/ncu.log 2>&1; echo ncu=$?
