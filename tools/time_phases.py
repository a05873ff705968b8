#!/usr/bin/env python3
"""Dev helper: average per-phase device times of K substeps on the bench
scene, ignoring step errors (used to time experimental library variants via
CKMPM_B200_LIB; a variant's physics may be wrong)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10399_b200 import abi  # noqa: E402
from paper_2412_10399_b200._lib import lib  # noqa: E402
from paper_2412_10399_b200.api import Simulation  # noqa: E402
from paper_2412_10399_b200.scene import block_scene, seed_particles  # noqa: E402

cells = int(os.environ.get("CELLS", "108"))
prec = int(os.environ.get("PREC", "8"))
fused = os.environ.get("FUSED", "1") == "1"
K = int(os.environ.get("STEPS", "10"))
model = os.environ.get("MODEL", "fixed_corotated")
scheme = os.environ.get("SCHEME", "apic")
kw = {"E": 1e4, "density": 1400.0, "boundary": "separate", "gravity": (0, -2.0, 0)} if model == "drucker_prager" else {}
cfg = block_scene(cells, model=model, scheme=scheme, kernel=os.environ.get("KERNEL", "compact"), **kw)
host = seed_particles(cfg, prec)
sim = Simulation(cfg, precision=prec, particles=host, fused=True if fused else False)
L = lib()
dt = sim.cfl_dt(1.0)
out = abi.StepOut()
for _ in range(3):
    L.ckg_step(sim._ctx, dt, C.byref(out))
acc = [0.0] * 6
rcs = set()
for _ in range(K):
    rcs.add(L.ckg_step(sim._ctx, dt, C.byref(out)))
    for k in range(6):
        acc[k] += out.phase_ms[k] / K
print(json.dumps({"lib": os.environ.get("CKMPM_B200_LIB", "default"), "fused": sim.fused(), "prec": prec,
                  "model": model, "scheme": scheme, "kernel": cfg.kernel, "n": len(host),
                  "phase_ms": dict(zip(abi.PHASE_NAMES, acc)), "total_ms": sum(acc), "rcs": sorted(rcs)}))
