"""Quadratic B-spline baseline (kernel.hpp:208-241,
transfer.hpp:285-320 / :512-543, grid.hpp:133-136): the 27-node kernel on the
unstaggered grid, against the reference engine run with kernel = quadratic
(oracle/_ref).  Bit-exact: active block set; tolerance: P2G node sums
<= 1e-13 of the field scale, particle state after 1 / 10 / 50 substeps
<= 1e-12 / 1e-10 / 1e-9."""
import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.scene import ConfigError, seed_particles
from tests.gpu_util import field_rel, gpu_sim, match_by_tag, nodes_by_coord, tag_volumes
from tests.util import perturb, small_scene

pytestmark = pytest.mark.gpu


def quad_scene(**kw):
    cfg = small_scene(**kw)
    cfg.kernel = "quadratic"
    return cfg


@pytest.mark.parametrize("scheme,model", [("pic", "fixed_corotated"), ("apic", "fixed_corotated"),
                                          ("apic", "drucker_prager"), ("apic", "j_fluid")])
def test_quad_p2g_nodes(scheme, model):
    cfg = quad_scene(scheme=scheme, model=model, res=32)
    p = perturb(seed_particles(cfg), seed=4, fscale=0.05, dx=1 / 32)
    dt = 2e-4
    rc, msg, rcoords, rnodes = bind.ref_p2g(cfg, p, dt)
    assert rc == 0, msg
    sim = gpu_sim(cfg, p)
    sim.step_phases(dt, abi.PHASE_P2G)
    gcoords, gnodes = sim.grid().blocks()
    G = nodes_by_coord(gcoords, gnodes)
    R = nodes_by_coord(rcoords, rnodes)
    assert set(G) == set(R)  # the quadratic footprint's active set, bit-exact
    a = np.stack([G[k] for k in R])
    b = np.stack([R[k] for k in R])
    for comp in range(4):
        scale = np.max(np.abs(b[..., comp]))
        err = np.max(np.abs(a[..., comp] - b[..., comp])) / scale
        assert err <= 1e-13, (comp, err)
    assert np.max(np.abs(a[:, 64:])) == 0.0  # grid slot 1 is unused


_FLOOR = {"x": 1.0, "v": 0.02, "F": 1.0, "B": 0.02 / 32 / 32, "J": 1.0}


@pytest.mark.parametrize("scheme,model,bc", [("pic", "fixed_corotated", "sticky"),
                                             ("apic", "fixed_corotated", "sticky"),
                                             ("apic", "drucker_prager", "separate"),
                                             ("apic", "j_fluid", "slip")])
def test_quad_state_after_n_steps(scheme, model, bc):
    cfg = quad_scene(scheme=scheme, model=model, bc=bc, res=32)
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=5, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    ref = bind.Ref(cfg, p0)
    sim = gpu_sim(cfg, p0)
    tol = {1: 1e-12, 10: 1e-10, 50: 1e-9}
    done = 0
    for target in (1, 10, 50):
        while done < target:
            dt = ref.cfl_dt(1.0)
            assert abs(dt - sim.cfl_dt(1.0)) <= 1e-9 * dt
            rc, msg = ref.step(dt)
            assert rc == 0, msg
            sim.step(dt)
            done += 1
        a, b = match_by_tag(sim.particles(), ref.particles())
        for f in ("x", "v", "F", "B", "J"):
            e = field_rel(a, b, f, floor=_FLOOR[f])
            assert e <= tol[target], (target, f, e)


def test_quad_frame_driver_matches_host_loop():
    cfg = quad_scene(res=32)
    p = tag_volumes(seed_particles(cfg))
    dev, host = gpu_sim(cfg, p), gpu_sim(cfg, p)
    for _ in range(2):
        assert dev.advance_frame() == host.advance_frame(device=False)
        assert dev.time() == host.time()
    a, b = match_by_tag(dev.particles(), host.particles())
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=_FLOOR[f]) <= 1e-10, f


def test_quad_mls_rejected_like_reference():
    cfg = quad_scene(scheme="mls", res=32)
    with pytest.raises(ConfigError, match="mls requires the compact kernel"):
        gpu_sim(cfg, seed_particles(small_scene(res=32)))


@pytest.mark.parametrize("kernel,per_p2g,per_g2p", [("quadratic", 27, 27), ("compact", 16, 16)])
def test_transfer_counters_per_kernel(kernel, per_p2g, per_g2p):
    """TransferCounters (transfer.hpp:32-45): the quadratic baseline visits 27
    nodes per particle in both transfers, the compact kernel 2 x 8 (acceptance
    criterion 7, tests/acceptance_main.cpp), through the host loop and the
    device frame driver alike."""
    cfg = small_scene(scheme="apic", res=32)
    cfg.kernel = kernel
    p = seed_particles(cfg)
    sim = gpu_sim(cfg, p)
    for _ in range(3):
        sim.step(sim.cfl_dt(1.0))
    c = sim.counters()
    assert c.p2g_node_visits == 3 * per_p2g * len(p)
    assert c.g2p_node_visits == 3 * per_g2p * len(p)
    sim.reset_counters()
    k = sim.advance_frame()
    c = sim.counters()
    assert k > 0
    assert c.p2g_node_visits == k * per_p2g * len(p)
    assert c.g2p_node_visits == k * per_g2p * len(p)
