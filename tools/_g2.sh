mkdir -p gpurun_out
KERNEL=quadratic timeout 300 python tools/time_phases.py > gpurun_out/r02_quad.json; cat gpurun_out/r02_quad.json
timeout 300 python tools/time_phases.py > gpurun_out/r02_compact.json; cat gpurun_out/r02_compact.json
timeout 900 python profiles/scenes.py > gpurun_out/r02_scenes.jsonl 2>&1; tail -5 gpurun_out/r02_scenes.jsonl
OUT=r02_launches bash tools/gpu_tasks.sh launches
NCUOUT=r02_full_10M NCU="p2g_tile|g2p_tile" SKIP=6 COUNT=2 bash tools/gpu_tasks.sh prof
NCUOUT=r02_full_10M_f32 NCU="p2g_tile|g2p_tile" SKIP=6 COUNT=2 BENCH_ARGS="--precision 4" bash tools/gpu_tasks.sh prof
