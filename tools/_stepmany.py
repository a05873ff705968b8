import ctypes as C, json, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2412_10399_b200 import abi
from paper_2412_10399_b200._lib import lib
from paper_2412_10399_b200.api import Simulation
from paper_2412_10399_b200.scene import block_scene, seed_particles
import torch
cells = int(os.environ.get("CELLS", "108"))
cfg = block_scene(cells)
host = seed_particles(cfg, 8)
sim = Simulation(cfg, precision=8, particles=host)
L = lib(); ctx = sim._ctx; dt = sim.cfl_dt(1.0); out = abi.StepOut()
for _ in range(5): assert L.ckg_step(ctx, dt, C.byref(out)) == 0
K = 20
for mode in ("loop", "many", "loop", "many"):
    torch.cuda.synchronize()
    L.ckg_timer_mark(ctx, 0)
    if mode == "loop":
        for _ in range(K): assert L.ckg_step(ctx, dt, C.byref(out)) == 0
    else:
        rc = L.ckg_step_many(ctx, dt, K, C.byref(out)); assert rc == 0, rc
        assert out.substeps_done == K
    L.ckg_timer_mark(ctx, 1)
    el = C.c_double(); L.ckg_timer_elapsed(ctx, 0, 1, C.byref(el))
    print(json.dumps({"mode": mode, "cells": cells, "ms_per_step": el.value / K, "launches": int(out.kernel_launches)}))
