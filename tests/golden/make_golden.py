"""Generate the committed golden fixtures from the REFERENCE engine itself
(oracle/_ref/libckref.so = /root/reference/proj/include/ckmpm compiled
unmodified with its Release flags).  Run in the build container:

    python tests/golden/make_golden.py

Each fixture scene_<name>.npz holds:
  config      JSON text of the scene (reference schema)
  p0          initial Particle<double> array (perturbed lattice, shuffled)
  dts         the cfl_dt schedule the reference took
  state_1, state_5   reference particle state after 1 and 5 substeps
  sort_keys, sort_order   reference stable sort of p0 (simulation.hpp:248-274)
  p2g_coords, p2g_nodes   reference grid after the first P2G (scatter_all,
                          deterministic), blocks sorted by coordinate
  active_1    active block coordinates after substep 1, sorted
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bind  # noqa: E402
from paper_2412_10399_b200.scene import SceneConfig, seed_particles  # noqa: E402

SCENES = {
    "fc_apic_sticky": {
        "resolution": 32, "scheme": "apic", "gravity": [0, -9.8, 0],
        "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1e5, "nu": 0.4}],
        "bodies": [{"shape": {"kind": "box", "lo": [0.375, 0.28125, 0.40625], "hi": [0.53125, 0.4375, 0.5625]},
                    "material": 0, "velocity": [0.3, -0.2, 0.1]}],
        "boundaries": [{"kind": "sticky", "lo": [0, 0, 0], "hi": [1, 0.25, 1]}]},
    "dp_apic_separate": {
        "resolution": 32, "scheme": "apic", "gravity": [0, -2.0, 0],
        "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 1e4, "nu": 0.4,
                       "friction_angle_deg": 30.0}],
        "bodies": [{"shape": {"kind": "sphere", "center": [0.5, 0.4, 0.5], "radius": 0.1}, "material": 0,
                    "velocity": [0, 0, 0.5]}],
        "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.28125, 1], "normal": [0, 1, 0]}]},
    "fluid_mls_slip": {
        "resolution": 32, "scheme": "mls", "gravity": [0, -9.8, 0],
        "materials": [{"model": "j_fluid", "density": 1000.0, "bulk": 1e4, "gamma": 7.0, "viscosity": 0.1}],
        "bodies": [{"shape": {"kind": "box", "lo": [0.40625, 0.3125, 0.40625], "hi": [0.5625, 0.46875, 0.5625]},
                    "material": 0}],
        "boundaries": [{"kind": "slip", "lo": [0, 0, 0], "hi": [1, 0.28125, 1], "normal": [0, 1, 0]}]},
    "fc_pic_nonpow2": {
        "resolution": 40, "scheme": "pic", "gravity": [0, 0, 0],
        "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1e5, "nu": 0.3}],
        "bodies": [{"shape": {"kind": "box", "lo": [0.35, 0.35, 0.35], "hi": [0.5, 0.475, 0.5]}, "material": 0,
                    "velocity": [-0.4, 0.25, 0.0]}],
        "boundaries": []},
}


def perturbed(p, res, seed):
    rng = np.random.default_rng(seed)
    q = p.copy()
    n = len(q)
    dx = 1.0 / res
    q["x"] = q["x"] + rng.uniform(-0.2, 0.2, (n, 3)) * dx
    q["v"] = q["v"] + rng.uniform(-0.02, 0.02, (n, 3))
    q["F"] = np.eye(3) + rng.uniform(-0.003, 0.003, (n, 3, 3))
    q["B"] = rng.uniform(-0.1, 0.1, (n, 3, 3)) * dx * dx
    q = q[rng.permutation(n)]
    return q


def sorted_blocks(coords, nodes):
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    return coords[order], nodes[order]


def main():
    for i, (name, obj) in enumerate(SCENES.items()):
        cfg = SceneConfig.from_json(obj)
        p0 = perturbed(seed_particles(cfg), cfg.resolution, 100 + i)
        keys, order = bind.ref_sort(cfg, p0)
        ref = bind.Ref(cfg, p0, threads=1, deterministic=True)
        dts = []
        states = {}
        active_1 = None
        for step in range(1, 6):
            dt = ref.cfl_dt(1.0)
            rc, msg = ref.step(dt)
            assert rc == 0, msg
            dts.append(dt)
            if step == 1:
                c, _ = ref.grid()
                active_1 = c[np.lexsort((c[:, 2], c[:, 1], c[:, 0]))]
            if step in (1, 5):
                states[step] = ref.particles()
        rc, msg, pc, pn = bind.ref_p2g(cfg, p0, dts[0])
        assert rc == 0, msg
        pc, pn = sorted_blocks(pc, pn)
        out = os.path.join(HERE, f"scene_{name}.npz")
        np.savez_compressed(out, config=json.dumps(obj), p0=p0, dts=np.array(dts), state_1=states[1],
                            state_5=states[5], sort_keys=keys, sort_order=order, p2g_coords=pc, p2g_nodes=pn,
                            active_1=active_1)
        print(f"{out}: {len(p0)} particles, {len(pc)} blocks, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
