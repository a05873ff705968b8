"""Fused G2P2G (csrc/ckg_g2p2g.cuh; CKG_FLAG_FUSED) for the
compact kernel with PIC/APIC on one GPU.  Parity against the C oracle and the
reference engine like the separate-kernel path, plus the mode's own
bookkeeping: the speculative next-substep scatter at the current dt (re-done
when the next dt differs), partial-phase calls, the grid facade after a fused
substep, and the equality of both paths."""
import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.api import Simulation
from paper_2412_10399_b200.scene import seed_particles
from tests.gpu_util import field_rel, match_by_tag, nodes_by_coord, tag_volumes
from tests.util import perturb, small_scene

pytestmark = pytest.mark.gpu

_FLOOR = {"x": 1.0, "v": 0.02, "F": 1.0, "B": 0.02 / 32 / 32, "J": 1.0}


def _state(scheme="apic", model="fixed_corotated", bc="sticky"):
    cfg = small_scene(scheme=scheme, model=model, bc=bc, res=32)
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=5, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    return cfg, p0


@pytest.mark.parametrize("scheme,model,bc,expect", [
    ("apic", "fixed_corotated", "sticky", True), ("pic", "fixed_corotated", "sticky", True),
    ("apic", "drucker_prager", "separate", True), ("apic", "j_fluid", "slip", True),
    ("mls", "fixed_corotated", "none", False)])
def test_mode_selection(scheme, model, bc, expect):
    cfg, p0 = _state(scheme, model, bc)
    with Simulation(cfg, particles=p0, fused=True) as s:
        assert s.fused() == expect
    with Simulation(cfg, particles=p0) as s:
        assert not s.fused()  # separate kernels by default
    cfg.kernel = "quadratic"
    if scheme != "mls":
        with Simulation(cfg, particles=p0, fused=True) as s:
            assert not s.fused()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("scheme,model,bc", [("pic", "fixed_corotated", "sticky"),
                                             ("apic", "fixed_corotated", "sticky"),
                                             ("apic", "drucker_prager", "separate"),
                                             ("apic", "j_fluid", "slip")])
def test_state_vs_oracle_both_modes(scheme, model, bc, fused):
    cfg, p0 = _state(scheme, model, bc)
    orc = bind.Oracle(cfg, p0)
    sim = Simulation(cfg, particles=p0, fused=fused)
    assert sim.fused() == fused
    tol = {1: 1e-12, 10: 1e-10, 100: 1e-8}
    done = 0
    for target in (1, 10, 100):
        while done < target:
            dt = orc.cfl_dt(1.0)
            assert abs(sim.cfl_dt(1.0) - dt) <= 1e-9 * dt
            rc, msg, _ = orc.step(dt)
            assert rc == 0, msg
            sim.step(dt)
            done += 1
        a, b = match_by_tag(sim.particles(), orc.particles())
        for f in ("x", "v", "F", "B", "J"):
            e = field_rel(a, b, f, floor=_FLOOR[f])
            assert e <= tol[target], (target, f, e)
    sim.close()


def test_changing_dt_redoes_the_speculative_scatter():
    """Every other substep at another dt: the speculative scatter (made at the
    previous dt) must be discarded and redone; the state follows the reference
    engine stepped with the same dt sequence."""
    cfg, p0 = _state()
    ref = bind.Ref(cfg, p0)
    sim = Simulation(cfg, particles=p0, fused=True)
    assert sim.fused()
    for k in range(30):
        dt = ref.cfl_dt(1.0) * (0.5 if k % 3 == 1 else 1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = match_by_tag(sim.particles(), ref.particles())
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=_FLOOR[f]) <= 1e-10, f
    sim.close()


def test_fused_equals_unfused_and_grid_facade():
    """Same substeps in both modes: state to round-off, and the grid facade
    after a completed substep (this substep's grid: mass and velocities after
    the grid update) identical in block set and values."""
    cfg, p0 = _state()
    a = Simulation(cfg, particles=p0, fused=True)
    b = Simulation(cfg, particles=p0)
    assert a.fused() and not b.fused()
    for _ in range(12):
        dt = b.cfl_dt(1.0)
        a.step(dt)
        b.step(dt)
    for f in ("x", "v", "F", "B", "J"):
        assert field_rel(a.particles(), b.particles(), f, floor=_FLOOR[f]) <= 1e-11, f
    ga, gb = a.grid(), b.grid()
    assert ga.active_block_count() == gb.active_block_count()
    A = nodes_by_coord(*ga.blocks())
    B = nodes_by_coord(*gb.blocks())
    assert set(A) == set(B)
    x = np.stack([A[k] for k in B])
    y = np.stack([B[k] for k in B])
    for comp in range(4):
        scale = max(np.max(np.abs(y[..., comp])), 1e-30)
        assert np.max(np.abs(x[..., comp] - y[..., comp])) <= 1e-11 * scale, comp
    for g in range(2):
        assert abs(ga.total_mass(g) - gb.total_mass(g)) <= 1e-12 * gb.total_mass(g)
    a.close()
    b.close()


def test_partial_phases_then_full_steps():
    """ckg_step_phases stops inside a substep (parity hooks); the fused mode's
    pools are rebuilt afterwards and the following substeps match the oracle."""
    cfg, p0 = _state()
    orc = bind.Oracle(cfg, p0)
    sim = Simulation(cfg, particles=p0, fused=True)
    for k in range(6):
        dt = orc.cfl_dt(1.0)
        if k in (0, 3):
            sim.step_phases(dt, abi.PHASE_P2G)
            sim.step_phases(dt, abi.PHASE_GRID)
        assert orc.step(dt)[0] == 0
        sim.step(dt)
    a, b = match_by_tag(sim.particles(), orc.particles())
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=_FLOOR[f]) <= 1e-11, f
    sim.close()


def test_upload_mid_run_discards_pending_scatter():
    """set_particles between substeps (the reference's mutable particles()):
    the pending scatter of the old state must not leak into the next substep."""
    cfg, p0 = _state()
    sim = Simulation(cfg, particles=p0, fused=True)
    orc = bind.Oracle(cfg, p0)
    dt = orc.cfl_dt(1.0)
    for _ in range(3):
        sim.step(dt)
        assert orc.step(dt)[0] == 0
    q = orc.particles()
    q["v"][:, 0] += 0.01
    sim.set_particles(q)
    orc2 = bind.Oracle(cfg, q)
    for _ in range(3):
        sim.step(dt)
        assert orc2.step(dt)[0] == 0
    a, b = match_by_tag(sim.particles(), orc2.particles())
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=_FLOOR[f]) <= 1e-11, f
    sim.close()


def test_fused_float_mode_vs_reference_float():
    cfg = small_scene(scheme="apic", res=32)
    p32 = seed_particles(cfg, 4)
    sim = Simulation(cfg, precision=4, particles=p32, fused=True)
    assert sim.fused()
    ref = bind.Ref(cfg, p32, precision=4)
    for _ in range(5):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = sim.particles(), ref.particles()
    assert np.array_equal(a["volume0"], b["volume0"])
    for f in ("x", "v", "F"):
        assert field_rel(a, b, f) <= 1e-5, f
    sim.close()
