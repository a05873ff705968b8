"""GPU parity on the layouts that exercise the transfer scheduling paths the
lattice ppc-8 scenes do not: dense blocks (ppc 27: 1728 particles per block,
several 512-particle P2G chunks, class counts of chunks past the first from
`ccnt`), jittered seeding (ppc 16: uneven class lists, shared base cells, the
rank-layer scatter), and mixed material models (the general G2P instance).
Same bars as tests/test_gpu_parity.py: P2G node sums <= 1e-13 of the field
scale, state after N substeps <= 1e-12 / 1e-10 relative."""
import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.scene import SceneConfig, seed_particles
from tests.gpu_util import field_rel, gpu_sim, match_by_tag, nodes_by_coord, tag_volumes
from tests.util import perturb, small_scene

pytestmark = pytest.mark.gpu

_FLOOR = {"x": 1.0, "v": 0.02, "F": 1.0, "B": 0.02 / 32 / 32, "J": 1.0}


def _p2g_matches(cfg, p, dt=2e-4):
    rc, msg, rcoords, rnodes = bind.ref_p2g(cfg, p, dt)
    assert rc == 0, msg
    sim = gpu_sim(cfg, p)
    sim.step_phases(dt, abi.PHASE_P2G)
    gcoords, gnodes = sim.grid().blocks()
    G = nodes_by_coord(gcoords, gnodes)
    R = nodes_by_coord(rcoords, rnodes)
    assert set(G) == set(R)
    a = np.stack([G[k] for k in R])
    b = np.stack([R[k] for k in R])
    for comp in range(4):
        scale = np.max(np.abs(b[..., comp]))
        err = np.max(np.abs(a[..., comp] - b[..., comp])) / scale
        assert err <= 1e-13, (comp, err)


def _steps_match(cfg, p0, steps=(1, 10)):
    orc = bind.Oracle(cfg, p0)
    sim = gpu_sim(cfg, p0)
    tol = {1: 1e-12, 10: 1e-10}
    done = 0
    for target in steps:
        while done < target:
            dt = orc.cfl_dt(1.0)
            rc, msg, _ = orc.step(dt)
            assert rc == 0, msg
            sim.step(dt)
            done += 1
        a, b = match_by_tag(sim.particles(), orc.particles())
        for f in ("x", "v", "F", "B", "J"):
            e = field_rel(a, b, f, floor=_FLOOR[f])
            assert e <= tol[target], (target, f, e)


@pytest.mark.parametrize("ppc", [27, 16])
@pytest.mark.parametrize("scheme", ["pic", "apic"])
def test_p2g_dense_and_jittered(ppc, scheme):
    cfg = small_scene(scheme=scheme, res=32, ppc=ppc)
    p = perturb(seed_particles(cfg), seed=7, fscale=0.05, dx=1 / 32)
    assert len(p) > 0
    _p2g_matches(cfg, p)


@pytest.mark.parametrize("ppc", [27, 16])
def test_state_dense_and_jittered(ppc):
    cfg = small_scene(scheme="apic", res=32, ppc=ppc)
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=8, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    _steps_match(cfg, p0)


def test_mixed_materials_general_instance():
    # an elastic block resting on a sand block: both models in one scene
    # select the general (all-model) G2P instance
    obj = {"name": "mixed", "resolution": 32, "scheme": "apic", "gravity": [0, -9.8, 0],
           "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1e5, "nu": 0.3},
                         {"model": "drucker_prager", "density": 1400.0, "E": 1e5, "nu": 0.3,
                          "friction_angle_deg": 30.0}],
           "bodies": [{"shape": {"kind": "box", "lo": [0.34375, 0.28125, 0.34375], "hi": [0.59375, 0.40625, 0.59375]},
                       "material": 1},
                      {"shape": {"kind": "box", "lo": [0.375, 0.40625, 0.375], "hi": [0.5625, 0.5625, 0.5625]},
                       "material": 0}],
           "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.25, 1], "normal": [0, 1, 0]}]}
    cfg = SceneConfig.from_json(obj)
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=9, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    _steps_match(cfg, p0)
