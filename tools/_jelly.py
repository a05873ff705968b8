import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_2412_10399_b200.api import Simulation
from paper_2412_10399_b200.scene import SceneConfig, seed_particles
from oracle import bind
obj = json.load(open("tests/golden/configs/jelly_cube.json"))
cfg = SceneConfig.from_json(obj)
print("frames", cfg.frames, "res", cfg.resolution, cfg.scheme)
p = seed_particles(cfg)
sim = Simulation(cfg, particles=p)
dts = []; ends = []
try:
    for f in range(cfg.frames):
        sim.advance_frame(lambda s, dt: dts.append(dt))
        ends.append(len(dts))
        if f % 20 == 0: print("compact frame", f, len(dts), sim.diagnostics().kinetic_energy, flush=True)
except Exception as e:
    print("compact failed at frame", f, len(dts), e)
    # reference for the same schedule
    ref = bind.Ref(cfg, p)
    for k, dt in enumerate(dts):
        rc, msg = ref.step(dt)
        if rc: print("ref failed", k, msg); break
    print("ref ok through", len(dts))
    sys.exit(0)
cfg.kernel = "quadratic"
q = Simulation(cfg, particles=p)
idx = 0
for f in range(cfg.frames):
    try:
        while idx < ends[f]:
            q.step(dts[idx]); idx += 1
    except Exception as e:
        print("quad failed at", idx, e); break
print("done")
