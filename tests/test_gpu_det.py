"""Deterministic mode (SimConfig::deterministic; the reference's serial
scatter, simulation.hpp:326-327, tests/test_sim.cpp:333-358): the device forms
every P2G node sum in a fixed order (csrc/ckg_transfer.cuh det_gather_kernel,
det_spill_kernel), so two runs from the same state are bitwise identical, and
the state still follows the reference engine to round-off."""
import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200.scene import seed_particles
from tests.gpu_util import field_rel, gpu_sim, match_by_tag, tag_volumes
from tests.util import perturb, small_scene

pytestmark = pytest.mark.gpu


def _scene(res, scheme="apic", model="fixed_corotated", bc="sticky"):
    cfg = small_scene(scheme=scheme, model=model, bc=bc, res=res)
    cfg.deterministic = True
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=11, fscale=0.01, vscale=0.05, bscale=0.1, xscale=0.3,
                             dx=1.0 / res))
    return cfg, p0


@pytest.mark.parametrize("res,scheme,model", [(32, "apic", "fixed_corotated"), (32, "pic", "fixed_corotated"),
                                              (32, "mls", "fixed_corotated"), (32, "apic", "drucker_prager"),
                                              (100, "apic", "fixed_corotated")])
def test_two_runs_bitwise_identical(res, scheme, model):
    cfg, p0 = _scene(res, scheme, model)
    runs = []
    for _ in range(2):
        sim = gpu_sim(cfg, p0)
        for _ in range(25):
            sim.step(sim.cfl_dt(1.0))
        runs.append(sim.particles())
        sim.close()
    assert runs[0].tobytes() == runs[1].tobytes()


@pytest.mark.parametrize("res", [32, 100])  # 100: non-power-of-two dx, out-of-tile records
def test_deterministic_state_vs_reference(res):
    cfg = small_scene(scheme="apic", res=res)
    cfg.deterministic = True
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=5, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.3,
                             dx=1.0 / res))
    ref = bind.Ref(cfg, p0, deterministic=True)
    sim = gpu_sim(cfg, p0)
    tol = {1: 1e-12, 10: 1e-10}
    for k in range(1, 11):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
        if k in tol:
            a, b = match_by_tag(sim.particles(), ref.particles())
            for f, fl in (("x", 1.0), ("v", 0.02), ("F", 1.0), ("B", 0.02 / res)):
                assert field_rel(a, b, f, floor=fl) <= tol[k], (k, f)


def test_deterministic_frames_bitwise():
    """advance_frame in deterministic mode (host loop; the CUDA-graph frame
    driver runs the atomic scatter) twice from the same state."""
    cfg = small_scene(scheme="apic", res=32, velocity=(0.3, -0.2, 0.1))
    cfg.deterministic = True
    p0 = seed_particles(cfg)
    out = []
    for _ in range(2):
        sim = gpu_sim(cfg, p0)
        for _ in range(2):
            sim.advance_frame()
        out.append(sim.particles())
        sim.close()
    assert out[0].tobytes() == out[1].tobytes()


def test_deterministic_moving_body_vs_reference():
    """A body sweeping across blocks (the active set and its slot numbering
    change every few substeps, leaving empty halo blocks in slots that held
    particles before): still the reference's state to round-off."""
    cfg = small_scene(scheme="apic", res=32, velocity=(0.3, 0.0, -0.2), bc="sticky")
    cfg.deterministic = True
    p0 = tag_volumes(seed_particles(cfg))
    ref = bind.Ref(cfg, p0, deterministic=True)
    sim = gpu_sim(cfg, p0)
    for _ in range(40):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = match_by_tag(sim.particles(), ref.particles())
    for f, fl in (("x", 1.0), ("v", 0.3), ("F", 1.0)):
        assert field_rel(a, b, f, floor=fl) <= 1e-10, f


def test_deterministic_flag_with_quadratic_baseline_matches_reference():
    """deterministic = true with kernel = quadratic: the baseline's P2G keeps
    its atomic flush (not bitwise reproducible), and the state still follows
    the reference engine."""
    cfg = small_scene(scheme="apic", res=32)
    cfg.kernel = "quadratic"
    cfg.deterministic = True
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=5, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    ref = bind.Ref(cfg, p0, deterministic=True)
    sim = gpu_sim(cfg, p0)
    for _ in range(10):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = match_by_tag(sim.particles(), ref.particles())
    for f, fl in (("x", 1.0), ("v", 0.02), ("F", 1.0)):
        assert field_rel(a, b, f, floor=fl) <= 1e-10, f
