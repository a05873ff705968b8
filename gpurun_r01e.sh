#!/bin/bash
# round-1e measurement set: parity suite, bench line, reference arm, launch list, ncu full (FP64 + FP32) of the transfer kernels at 10M
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
OUT=launches_r01e ./gpurun_launches.sh
CELLS=108 NCUOUT=r01e_full_10M ./gpurun_prof.sh
CELLS=108 NCUOUT=r01e_full_10M_f32 BENCH_ARGS="--precision 4 --no-single" ./gpurun_prof.sh
ls -la gpurun_out/
