import os, sys, json
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2412_10399_b200.api import Simulation
from paper_2412_10399_b200.scene import SceneConfig, seed_particles
from oracle import bind
from tests.gpu_util import field_rel, match_by_tag, tag_volumes
obj = json.load(open("tests/golden/configs/jelly_cube.json"))
cfg = SceneConfig.from_json(obj)
p = tag_volumes(seed_particles(cfg))
sim = Simulation(cfg, particles=p)
ref = bind.Ref(cfg, p)
for k in range(700):
    dt = ref.cfl_dt(1.0)
    gdt = sim.cfl_dt(1.0)
    rc, msg = ref.step(dt)
    if rc: print("ref fail", k, msg); break
    try:
        sim.step(dt)
    except Exception as e:
        print("gpu fail", k, e); break
    if k % 25 == 0 or k > 630:
        a, b = match_by_tag(sim.particles(), ref.particles())
        errs = {f: field_rel(a, b, f, floor=fl) for f, fl in (("x", 1.0), ("v", 0.5), ("F", 1.0))}
        dF = np.linalg.det(a["F"]); dFr = np.linalg.det(b["F"])
        print(k, dt, abs(gdt - dt) / dt, errs, "minJ gpu", dF.min(), "ref", dFr.min(), flush=True)
