#!/usr/bin/env python3
"""Throughput on the BASELINE.json scene family (SURVEY Appendix C JSON),
one B200, FP64: device-resident substeps at the replayed t=0 dt (as bench.py),
and whole frames through advance_frame -- the device frame driver (one CUDA
graph per frame) against the host loop over ckg_step.  Measurement helper,
prints one line per scene; run with a GPU (gpurun)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
from paper_2412_10399_b200.api import Simulation  # noqa: E402
from paper_2412_10399_b200.scene import SceneConfig  # noqa: E402

SCENES = {
    "C1b_jelly_110k": {"name": "C1b_jelly_110k", "resolution": 64, "scheme": "apic", "gravity": [0, -9.8, 0], "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 100000.0, "nu": 0.4}], "bodies": [{"shape": {"kind": "box", "lo": [0.3125, 0.3125, 0.3125], "hi": [0.6875, 0.6875, 0.6875]}, "material": 0, "ppc": 8}], "boundaries": [{"kind": "sticky", "lo": [0, 0, 0], "hi": [1, 0.0625, 1]}]},
    "C2_two_spheres_1M": {"name": "C2_two_spheres_1M", "resolution": 256, "scheme": "apic", "gravity": [0, 0, 0], "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1000000.0, "nu": 0.4}], "bodies": [{"shape": {"kind": "sphere", "center": [0.125, 0.125, 0.125], "radius": 0.09765625}, "material": 0, "ppc": 8, "velocity": [0.05, 0.05, 0.05]}, {"shape": {"kind": "sphere", "center": [0.5, 0.5, 0.5], "radius": 0.09765625}, "material": 0, "ppc": 8, "velocity": [-0.05, -0.05, -0.05]}], "boundaries": []},
    "C3_sand_column_4M": {"name": "C3_sand_column_4M", "resolution": 256, "scheme": "apic", "gravity": [0, -2.0, 0], "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 10000.0, "nu": 0.4, "friction_angle_deg": 30.0}], "bodies": [{"shape": {"kind": "box", "lo": [0.375, 0.0625, 0.375], "hi": [0.625, 0.5625, 0.625]}, "material": 0, "ppc": 8}], "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]},
    "C4_sandcastle_10M": {"name": "C4_sandcastle_10M", "resolution": 512, "scheme": "apic", "gravity": [0, -0.1, 0], "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 10000.0, "nu": 0.4, "friction_angle_deg": 30.0}, {"model": "fixed_corotated", "density": 1000.0, "E": 10000000.0, "nu": 0.2}], "bodies": [{"shape": {"kind": "box", "lo": [0.40625, 0.0625, 0.39453125], "hi": [0.6171875, 0.2734375, 0.60546875]}, "material": 0, "ppc": 8}, {"shape": {"kind": "sphere", "center": [0.35625, 0.16796875, 0.5], "radius": 0.01953125}, "material": 1, "ppc": 8, "velocity": [10.0, 0, 0]}], "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]},
}


def run(name, frames, steps, frame_dt=None):
    obj = dict(SCENES[name])
    if frame_dt:
        obj["frame_dt"] = frame_dt
    cfg = SceneConfig.from_json(obj)
    row = {"scene": name}
    # device-resident substeps at the replayed t=0 dt
    sim = Simulation(cfg)
    n = sim._n
    row["particles"] = n
    dt = sim.cfl_dt(1.0)
    for _ in range(3):
        sim.step(dt)
    sim.reset_timers()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step(dt)
    wall = time.perf_counter() - t0
    dev = sim.timers().total()
    row["step_device_ms"] = dev / steps * 1e3
    row["step_wall_ms"] = wall / steps * 1e3
    row["p_substeps_per_s_device"] = n * steps / dev
    # the same substeps through step_many (one frame-graph launch, fixed dt)
    sim.step_many(dt, steps)  # warm-up (graph instantiation)
    t0 = time.perf_counter()
    sim.step_many(dt, steps)
    wall = time.perf_counter() - t0
    row["step_many_wall_ms"] = wall / steps * 1e3
    row["p_substeps_per_s_step_many"] = n * steps / wall
    sim.close()
    # frames: device driver vs host loop (same start state, warm-up frame first)
    for mode in ("device", "host"):
        s = Simulation(cfg)
        s.advance_frame(device=(mode == "device"))
        t0 = time.perf_counter()
        subs = 0
        for _ in range(frames):
            subs += s.advance_frame(device=(mode == "device"))
        wall = time.perf_counter() - t0
        row[f"frame_{mode}_ms"] = wall / frames * 1e3
        row[f"frame_{mode}_substeps"] = subs / frames
        row[f"p_substeps_per_s_{mode}_loop"] = n * subs / wall
        s.close()
    return row


if __name__ == "__main__":
    plan = [("C1b_jelly_110k", 10, 50, None), ("C2_two_spheres_1M", 5, 30, 1.0 / 600),
            ("C3_sand_column_4M", 3, 20, 1.0 / 60), ("C4_sandcastle_10M", 2, 10, 1.0 / 6000)]
    only = sys.argv[1:]
    for name, frames, steps, fdt in plan:
        if only and name not in only:
            continue
        print(json.dumps(run(name, frames, steps, fdt)), flush=True)
