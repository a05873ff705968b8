#!/usr/bin/env python3
"""Per-substep cost of the x-slab path on one GPU: the C5 block
run as 1 slab (no neighbours: the slab bookkeeping alone) and as 2 slabs in
loopback (exchanges as device copies), against the single-domain ckg_step.
Measurement helper (wall time with device sync per substep)."""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import torch  # noqa: E402

from paper_2412_10399_b200.api import Simulation  # noqa: E402
from paper_2412_10399_b200.scene import block_scene  # noqa: E402
from paper_2412_10399_b200.slab import build_ranks, run_loopback  # noqa: E402


def main(cells=108, steps=10):
    cfg = block_scene(cells)
    sim = Simulation(cfg)
    dt = sim.cfl_dt(1.0)
    for _ in range(3):
        sim.step(dt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step(dt)
    single = (time.perf_counter() - t0) / steps * 1e3
    n = sim._n
    sim.close()
    row = {"particles": n, "single_domain_ms": single}
    for world in (1, 2):
        _, ranks = build_ranks(cfg, world)
        for _ in range(3):
            run_loopback(ranks, dt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            run_loopback(ranks, dt)
        torch.cuda.synchronize()
        row[f"slab{world}_loopback_ms"] = (time.perf_counter() - t0) / steps * 1e3
        for r in ranks:
            r.close()
    print(json.dumps(row))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 108)
