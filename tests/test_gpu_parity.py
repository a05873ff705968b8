"""GPU parity vs the reference engine / C oracle, through the C-ABI.

Bit-exact: block keys, stable sorted order, the 6 stencil bases, the active
block set (SURVEY §8c parity protocol).  Tolerance: P2G node sums <= 1e-13
relative to the field scale (test_transfer.cpp:139-141); particle state after
1 / 10 / 100 substeps <= 1e-12 / 1e-10 / 1e-8 relative (north star: float
atomics reorder sums)."""
import ctypes as C
import glob
import os

import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.scene import (InvertedElementError, NumericalError, OutOfDomainError,
                                         SceneConfig, seed_particles)
from tests.gpu_util import field_rel, gpu_sim, match_by_tag, nodes_by_coord, tag_volumes
from tests.util import perturb, small_scene

pytestmark = pytest.mark.gpu


def _shuffled(p, seed=0):
    return p[np.random.default_rng(seed).permutation(len(p))]


def _adversarial(res, n=20000, seed=0):
    """Positions on and next to quarter-cell / block boundaries at a
    non-power-of-two resolution (where the multiply- and divide-form bin
    formulas can disagree)."""
    obj = {"resolution": res, "scheme": "apic", "materials": [{"model": "fixed_corotated", "density": 1000.0,
                                                                "E": 1e5, "nu": 0.3}],
           "bodies": [{"shape": {"kind": "box", "lo": [0.3, 0.3, 0.3], "hi": [0.4, 0.4, 0.4]}, "material": 0}]}
    cfg = SceneConfig.from_json(obj)
    dx = cfg.dx()
    rng = np.random.default_rng(seed)
    cells = rng.integers(3, res - 4, (n, 3)).astype(np.float64)
    frac = rng.choice([0.0, 0.25, 0.5, 0.75, 1.0], (n, 3))
    ulps = rng.integers(-3, 4, (n, 3))
    x = (cells + frac) * dx
    x = x + ulps * np.spacing(x)
    p = np.zeros(n, dtype=abi.particle_dtype(8))
    p["x"] = x
    p["F"] = np.eye(3)
    p["J"] = 1.0
    p["mass"] = 1.0
    p["volume0"] = dx ** 3 / 8
    return cfg, p


@pytest.mark.parametrize("res", [32, 96, 100, 200])
def test_binning_bitwise(res):
    if res == 32:
        cfg = small_scene(res=32)
        p = _shuffled(perturb(seed_particles(cfg), seed=1, xscale=1.5, dx=1 / 32))
    else:
        cfg, p = _adversarial(res, seed=res)
    k_ref, o_ref = bind.ref_sort(cfg, p)
    sim = gpu_sim(cfg, p)
    k_gpu, o_gpu = sim.debug_sort()
    assert np.array_equal(k_gpu, k_ref)
    assert np.array_equal(o_gpu, o_ref)
    # stencil bases, both grids (kernel.hpp:114-120), vs the reference axis_pair
    bases = sim.debug_bases()
    r = bind.ref_lib()
    b = C.c_int32()
    v = (C.c_double * 5)()
    dx = cfg.dx()
    idx = np.random.default_rng(res).choice(len(p), min(len(p), 3000), replace=False)
    for i in idx:
        for g, k in ((0, -1), (1, 1)):
            for a in range(3):
                r.ckref_axis_pair(float(p["x"][i, a]), k, float(dx), C.byref(b), v)
                assert bases[i, g, a] == b.value


def test_activation_set_bitwise():
    cfg = small_scene(res=32)
    p = perturb(seed_particles(cfg), seed=3, xscale=1.0, dx=1 / 32)
    ref = bind.Ref(cfg, p)
    assert ref.step(1e-5)[0] == 0
    rc, _ = ref.grid()
    sim = gpu_sim(cfg, p)
    sim.step_phases(1e-5, abi.PHASE_ACTIVATE)
    gc, _ = sim.grid().blocks()
    assert sim.grid().active_block_count() == len(rc)
    assert set(map(tuple, gc)) == set(map(tuple, rc))


@pytest.mark.parametrize("scheme", ["pic", "apic", "mls"])
@pytest.mark.parametrize("model", ["fixed_corotated", "drucker_prager", "j_fluid"])
def test_p2g_nodes(scheme, model):
    cfg = small_scene(scheme=scheme, model=model, res=32)
    p = perturb(seed_particles(cfg), seed=4, fscale=0.05, dx=1 / 32)
    dt = 2e-4
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


# Field scales below which differences are round-off of a vanishing field:
# x ~ 1, v ~ 0.05 m/s, B ~ v dx^2-ish, F ~ 1.
_FLOOR = {"x": 1.0, "v": 0.02, "F": 1.0, "B": 0.02 / 32 / 32, "J": 1.0}

STEP_CASES = [
    ("pic", "fixed_corotated", "sticky"),
    ("apic", "fixed_corotated", "sticky"),
    ("mls", "fixed_corotated", "none"),
    ("apic", "drucker_prager", "separate"),
    ("apic", "j_fluid", "slip"),
]


@pytest.mark.parametrize("scheme,model,bc", STEP_CASES)
def test_state_after_n_steps(scheme, model, bc):
    cfg = small_scene(scheme=scheme, model=model, bc=bc, res=32)
    # mild perturbation: every transfer term is exercised but the body stays
    # well inside the elastic regime for 100 substeps
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=5, fscale=0.003, vscale=0.02, bscale=0.1, xscale=0.05,
                             dx=1 / 32))
    orc = bind.Oracle(cfg, p0)
    sim = gpu_sim(cfg, p0)
    tol = {1: 1e-12, 10: 1e-10, 100: 1e-8}
    done = 0
    for target in (1, 10, 100):
        while done < target:
            dt = orc.cfl_dt(1.0)
            gdt = sim.cfl_dt(1.0)
            assert abs(dt - gdt) <= 1e-9 * dt
            rc, msg, _ = orc.step(dt)
            assert rc == 0, msg
            sim.step(dt)
            done += 1
        a, b = match_by_tag(sim.particles(), orc.particles())
        for f in ("x", "v", "F", "B", "J"):
            e = field_rel(a, b, f, floor=_FLOOR[f])
            assert e <= tol[target], (target, f, e)


def test_momentum_conservation_matches_reference_level():
    # force-free colliding blocks: total momentum must stay at round-off
    cfg = small_scene(scheme="apic", res=48, bc="none", gravity=(0, 0, 0), lo=(0.3, 0.3, 0.3),
                      hi=(0.45, 0.45, 0.45), velocity=(0.3, -0.2, 0.1), E=1e4)
    p = seed_particles(cfg)
    sim = gpu_sim(cfg, p)
    d0 = sim.diagnostics()
    for _ in range(100):
        sim.step(sim.cfl_dt(1.0))
    d1 = sim.diagnostics()
    pscale = float(np.sum(p["mass"]) * np.max(np.abs(p["v"])))
    assert np.max(np.abs(d1.momentum - d0.momentum)) <= 1e-12 * pscale


def test_out_of_domain_error_identifies_particle():
    cfg = small_scene(res=32)
    p = seed_particles(cfg)
    p["x"][5, 0] = 1.5 / 32
    ref = bind.Ref(cfg, p)
    rc, msg = ref.step(1e-4)
    sim = gpu_sim(cfg, p)
    with pytest.raises(OutOfDomainError) as ei:
        sim.step(1e-4)
    assert str(ei.value) == msg
    assert ei.value.particle_index == int(msg.split()[1])


@pytest.mark.parametrize("field", ["v", "x"])
def test_nonfinite_state_aborts_loudly(field):
    """test_sim.cpp:412-417: a NaN in the state aborts the step with a
    NumericalError; the GPU raises the same type and message as the
    reference for the same input."""
    cfg = small_scene(res=32)
    p = seed_particles(cfg)
    p[field][10, 1] = np.nan
    rc, msg = bind.Ref(cfg, p).step(1e-4)
    assert rc == 3
    sim = gpu_sim(cfg, p)
    with pytest.raises(NumericalError) as ei:
        sim.step(1e-4)
    assert str(ei.value) == msg


def test_inverted_element_raises():
    cfg = small_scene(res=32)
    p = seed_particles(cfg)
    p["F"][3] = np.diag([1.0, 1.0, -1.0])
    sim = gpu_sim(cfg, p)
    with pytest.raises(InvertedElementError, match="fixed corotated stress: det F <= 0"):
        sim.step(1e-4)


def test_float_mode_vs_reference_float():
    cfg = small_scene(scheme="apic", res=32)
    p32 = seed_particles(cfg, 4)
    k_ref, o_ref = bind.ref_sort(cfg, p32, precision=4)
    sim = gpu_sim(cfg, p32, precision=4)
    k, o = sim.debug_sort()
    assert np.array_equal(k, k_ref) and np.array_equal(o, o_ref)
    ref = bind.Ref(cfg, p32, precision=4)
    for _ in range(3):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = sim.particles(), ref.particles()
    for f in ("x", "v", "F"):
        assert field_rel(a, b, f) <= 1e-5, f


def test_step_many_equals_single_steps():
    cfg = small_scene(scheme="apic", res=32)
    p = seed_particles(cfg)
    s1 = gpu_sim(cfg, p)
    s2 = gpu_sim(cfg, p)
    dt = s1.cfl_dt(1.0)
    for _ in range(5):
        s1.step(dt)
    s2.step_many(dt, 5)
    a, b = s1.particles(), s2.particles()
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=1e-3) <= 1e-12, f


def test_step_many_graph_path_equals_single_steps():
    """After a first substep (stored-order keys and stress cache in place)
    step_many runs its substeps as one launch of the frame graph in fixed-dt
    mode; the state equals single steps, odd and even counts."""
    cfg = small_scene(scheme="apic", res=32)
    p = seed_particles(cfg)
    s1 = gpu_sim(cfg, p)
    s2 = gpu_sim(cfg, p)
    dt = s1.cfl_dt(1.0)
    for _ in range(14):
        s1.step(dt)
    s2.step(dt)
    s2.step(dt)  # (an incremental sort: its crosser count lets the graph path in)
    s2.step_many(dt, 5)
    s2.step_many(dt, 7)
    assert s2.step_count() == 14
    a, b = s1.particles(), s2.particles()
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=1e-3) <= 1e-12, f


def test_stored_order_tracks_reference_sort():
    """Bodies moving across block boundaries every substep: the device's
    stored particle order (its incremental stable sort, ckg_isort.cuh) must
    equal the reference's full stable counting sort after every substep."""
    cfg = small_scene(scheme="apic", res=32, bc="none", gravity=(0, 0, 0), velocity=(2.0, -1.5, 1.0))
    p0 = tag_volumes(perturb(seed_particles(cfg), seed=9, fscale=0.002, vscale=0.01, bscale=0.05,
                             xscale=0.2, dx=1 / 32))
    p0 = p0[np.random.default_rng(1).permutation(len(p0))]  # unsorted start -> full radix first
    ref = bind.Ref(cfg, p0)
    sim = gpu_sim(cfg, p0)
    kinds = set()
    for step in range(40):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
        kinds.add(sim.last_sort_kind())
        a, b = sim.particles(), ref.particles()
        assert np.array_equal(a["volume0"], b["volume0"]), f"order diverged at step {step}"
    assert 2 in kinds, "incremental merge path not exercised"


GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "scene_*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[6:-4] for p in GOLDEN])
def test_device_vs_golden(path):
    """Device path against fixtures produced by the reference engine itself
    (no /root/reference needed at run time)."""
    import json as _json
    z = np.load(path, allow_pickle=False)
    cfg = SceneConfig.from_json(_json.loads(str(z["config"])))
    p0 = z["p0"]
    sim = gpu_sim(cfg, p0)
    k, o = sim.debug_sort()
    assert np.array_equal(k, z["sort_keys"]) and np.array_equal(o, z["sort_order"])
    sim.step_phases(float(z["dts"][0]), abi.PHASE_P2G)
    gc, gn = sim.grid().blocks()
    order = np.lexsort((gc[:, 2], gc[:, 1], gc[:, 0]))
    gc, gn = gc[order], gn[order]
    # P2G pass covers the active set; the reference lists the same set
    assert np.array_equal(gc, z["p2g_coords"])
    for comp in range(4):
        ref = z["p2g_nodes"][..., comp]
        assert np.max(np.abs(gn[..., comp] - ref)) <= 1e-13 * np.max(np.abs(ref)), comp
    tol = {1: 1e-12, 5: 1e-11}
    for step, dt in enumerate(z["dts"], start=1):
        assert abs(sim.cfl_dt(1.0) - dt) <= 1e-12 * dt
        sim.step(float(dt))
        if step in tol:
            a, b = sim.particles(), z[f"state_{step}"]
            for f, fl in (("x", 1.0), ("v", 0.1), ("F", 1.0), ("B", 1e-4), ("J", 1.0)):
                x = np.asarray(a[f], dtype=np.float64)
                y = np.asarray(b[f], dtype=np.float64)
                err = float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), fl))
                assert err <= tol[step], (step, f, err)


def test_step_many_stops_at_failing_substep():
    """A substep that throws leaves the state of the last completed one
    (the reference's step() loop): a block flying into the domain inset raises
    OutOfDomainError inside step_many after some substeps; the state and
    step count equal those of the same number of single step() calls."""
    cfg = small_scene(scheme="apic", res=32, bc="none", gravity=(0, 0, 0), lo=(0.0625 + 0.01, 0.4, 0.4),
                      hi=(0.0625 + 0.09, 0.48, 0.48), velocity=(-3.0, 0.0, 0.0))
    p = seed_particles(cfg)
    dt = 1e-3  # 3 m/s * 1 ms = ~0.1 cell per substep
    s1 = gpu_sim(cfg, p)
    k_ok = 0
    with pytest.raises(OutOfDomainError):
        for _ in range(200):
            s1.step(dt)
            k_ok += 1
    assert 2 < k_ok < 200
    s2 = gpu_sim(cfg, p)
    with pytest.raises(OutOfDomainError):
        s2.step_many(dt, k_ok + 5)
    assert s2.step_count() == k_ok
    a, b = s1.particles(), s2.particles()
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=1e-3) <= 1e-12, f
    # the same through the graph path (one single step first)
    s3 = gpu_sim(cfg, p)
    s3.step(dt)
    s3.step(dt)
    with pytest.raises(OutOfDomainError) as ei:
        s3.step_many(dt, k_ok + 5)
    assert s3.step_count() == k_ok
    c = s3.particles()
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, c, f, floor=1e-3) <= 1e-12, f
    # and stepping on from the restored state works
    s3.set_particles(s1.particles())


def test_empty_and_single_particle_states():
    """Edge cases of the particle count: an empty state steps (no work, the
    step counter advances as in the reference's loop over zero particles) and
    a single particle follows the reference engine."""
    cfg = small_scene(scheme="apic", res=32)
    p = seed_particles(cfg)
    sim = gpu_sim(cfg, p)
    sim.set_particles(p[:0])
    assert len(sim.particles()) == 0
    sim.step(1e-4)
    sim.step_many(1e-4, 3)
    assert len(sim.particles()) == 0
    one = tag_volumes(p[len(p) // 2:len(p) // 2 + 1].copy())
    ref = bind.Ref(cfg, one)
    sim.set_particles(one)
    for _ in range(5):
        dt = ref.cfl_dt(1.0)
        assert ref.step(dt)[0] == 0
        sim.step(dt)
    a, b = sim.particles(), ref.particles()
    assert len(a) == 1
    for f in ("x", "v", "F", "B"):
        assert field_rel(a, b, f, floor=1e-3) <= 1e-12, f
