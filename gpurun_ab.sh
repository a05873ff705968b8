#!/bin/bash
# A/B of build/var variants, then the GPU parity suite on the default library
REPS=1 bash gpurun_var.sh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
