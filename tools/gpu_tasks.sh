#!/bin/bash
# Dev helper run on the GPU box through gpurun:  bash tools/gpu_tasks.sh TASK...
#   check     the GPU parity suite (-m gpu), smoke(), the default bench line
#   tests     the GPU parity suite only (PYTEST_ARGS to filter)
#   bench     the default bench line (BENCH_ARGS appended)
#   ref       the reference arm (bench.py --impl reference)
#   launches  per-launch device times of the bench command (ncu launch list -> gpurun_out/$OUT.csv)
#   prof      ncu --set full of the transfer kernels (NCU regex, SKIP, COUNT, CELLS) -> gpurun_out/$NCUOUT.ncu-rep
mkdir -p gpurun_out
for task in "$@"; do
case $task in
  check|tests)
    timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
    tail -15 gpurun_out/pytest_gpu.log
    if [ $task = check ]; then
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
      timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -c 4000 gpurun_out/bench_full.log
    fi ;;
  bench)
    timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${OUT:-full}.log 2>&1; echo bench=$?; tail -c 4000 gpurun_out/bench_${OUT:-full}.log ;;
  ref)
    timeout 900 python bench.py --impl reference ${REF_ARGS} > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -c 2000 gpurun_out/bench_ref.log ;;
  launches)
    cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-chains 1 --no-single ${BENCH_ARGS}"
    $cmd > gpurun_out/plain.log 2>&1; echo plain=$?
    ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-400} --csv --log-file gpurun_out/${OUT:-launches}.csv $cmd > gpurun_out/ncu_launch.log 2>&1; echo ncu=$? ;;
  prof)
    cmd="python bench.py --cells ${CELLS:-108} --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-chains 1 --no-single ${BENCH_ARGS}"
    $cmd > gpurun_out/plain_prof.log 2>&1; echo plain=$?
    ncu --set full --clock-control none --import-source on -k regex:"${NCU:-p2g_tile|g2p_tile}" -s ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/${NCUOUT:-prof} -f $cmd > gpurun_out/ncu.log 2>&1; echo ncu=$? ;;
  *) echo "unknown task $task" ;;
esac
done
