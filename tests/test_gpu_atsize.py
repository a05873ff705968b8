"""GPU parity against the reference engine itself at BASELINE's sizes.

The device path (C-ABI) and the reference `ckmpm::Simulation<T>` (oracle/_ref,
the unmodified headers, stepped on all host cores in its default atomic mode)
are fed the same particle array and the same dt sequence and compared:

* C5_block_108 (10,077,696 FC particles, res 512; the bench workload):
  block keys and stable order bit-exact vs the reference's own
  `sort_particles` (simulation.hpp:248-274); stored order equal after every
  substep; x, v, F, B after 1 and 3 substeps <= 1e-12 / 1e-11.
* C2_two_spheres_1M (1,047,968 p, north-star config 2): total and mass-free
  momentum vs the reference over 20 substeps; state <= 1e-10.
* C3_sand_column_4M (4,194,304 DP particles) and C4_sandcastle_10M
  (10,111,224 p, DP block + fast FC ball): 3 substeps each.
* twisting_bar_ppc8 (the reference's own config, rotating sticky BCs
  v0 + omega x (x - c), grid.hpp:38-44): 50 substeps.
* a clamp_singular scene (transfer.hpp:574-577 + material clamp): 10 substeps.

Particles are matched positionally: both engines keep the reference's stored
order (checked bit-exactly through a per-particle tag in volume0, which every
engine carries unchanged).  Float atomics reorder sums in both engines, so
state agrees to round-off, not bitwise.
"""
import os

import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200.api import Simulation
from paper_2412_10399_b200.scene import SceneConfig, block_scene, seed_particles
from tests.gpu_util import field_rel, tag_volumes

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1

# SURVEY Appendix C scene JSON (reference schema, io.hpp:242-315)
C2 = {"name": "C2_two_spheres_1M", "resolution": 256, "scheme": "apic", "gravity": [0, 0, 0],
      "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1000000.0, "nu": 0.4}],
      "bodies": [{"shape": {"kind": "sphere", "center": [0.125, 0.125, 0.125], "radius": 0.09765625},
                  "material": 0, "ppc": 8, "velocity": [0.05, 0.05, 0.05]},
                 {"shape": {"kind": "sphere", "center": [0.5, 0.5, 0.5], "radius": 0.09765625},
                  "material": 0, "ppc": 8, "velocity": [-0.05, -0.05, -0.05]}],
      "boundaries": []}
C3 = {"name": "C3_sand_column_4M", "resolution": 256, "scheme": "apic", "gravity": [0, -2.0, 0],
      "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 10000.0, "nu": 0.4,
                     "friction_angle_deg": 30.0}],
      "bodies": [{"shape": {"kind": "box", "lo": [0.375, 0.0625, 0.375], "hi": [0.625, 0.5625, 0.625]},
                  "material": 0, "ppc": 8}],
      "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]}
C4 = {"name": "C4_sandcastle_10M", "resolution": 512, "scheme": "apic", "gravity": [0, -0.1, 0],
      "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 10000.0, "nu": 0.4,
                     "friction_angle_deg": 30.0},
                    {"model": "fixed_corotated", "density": 1000.0, "E": 10000000.0, "nu": 0.2}],
      "bodies": [{"shape": {"kind": "box", "lo": [0.40625, 0.0625, 0.39453125],
                            "hi": [0.6171875, 0.2734375, 0.60546875]}, "material": 0, "ppc": 8},
                 {"shape": {"kind": "sphere", "center": [0.35625, 0.16796875, 0.5], "radius": 0.01953125},
                  "material": 1, "ppc": 8, "velocity": [10.0, 0, 0]}],
      "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]}
# proj/configs/twisting_bar_ppc8.json (scene part)
TWIST = {"name": "twisting_bar_ppc8", "resolution": 64, "extent": 1.0, "kernel": "compact", "scheme": "apic",
         "gravity": [0.0, 0.0, 0.0], "cfl": 0.5, "frame_dt": 0.020833333333333332,
         "materials": [{"model": "fixed_corotated", "density": 2.0, "E": 100.0, "nu": 0.4}],
         "bodies": [{"shape": {"kind": "box", "lo": [0.25, 0.4375, 0.4375], "hi": [0.75, 0.5625, 0.5625]},
                     "material": 0, "ppc": 8}],
         "boundaries": [{"kind": "sticky", "lo": [0.234375, 0.40625, 0.40625], "hi": [0.296875, 0.59375, 0.59375],
                         "velocity": [0.0, 0.0, 0.0], "omega": [1.0, 0.0, 0.0], "center": [0.265625, 0.5, 0.5]},
                        {"kind": "sticky", "lo": [0.703125, 0.40625, 0.40625], "hi": [0.765625, 0.59375, 0.59375],
                         "velocity": [0.0, 0.0, 0.0], "omega": [-1.0, 0.0, 0.0], "center": [0.734375, 0.5, 0.5]}]}

# natural field scales (a vanishing field is judged against these floors);
# B (APIC affine velocity, ~ v dx) is judged against max|v| dx of the
# reference state: its error enters the next P2G as B D^-1 xi ~ B / dx, i.e.
# as a velocity error (a translating body's B is pure round-off)
FLOOR = {"x": 1.0, "v": 0.01, "F": 1.0, "B": None, "J": 1.0}


def _run_pair(cfg, p0, steps, tol, fields=("x", "v", "F", "B"), threads=THREADS, deterministic=False,
              floors=FLOOR, each=None):
    """Step the device and the reference side by side with the reference's dt
    sequence (cfl_dt(1) before each substep, asserted equal on both sides);
    compare the stored order (tag) after every substep and the state at the
    substeps named in `tol`."""
    p0 = tag_volumes(p0)
    ref = bind.Ref(cfg, p0, threads=threads, deterministic=deterministic)
    errs = {}
    with Simulation(cfg, precision=8, particles=p0) as sim:
        for k in range(1, steps + 1):
            dt = ref.cfl_dt(1.0)
            assert abs(sim.cfl_dt(1.0) - dt) <= 1e-9 * dt, k
            rc, msg = ref.step(dt)
            assert rc == 0, msg
            sim.step(dt)
            if each is not None:
                each(k, sim, ref)
            if k in tol or k == steps:
                a, b = sim.particles(), ref.particles()
                assert np.array_equal(a["volume0"], b["volume0"]), f"stored order differs after substep {k}"
                if k in tol:
                    for f in fields:
                        fl = floors[f]
                        if fl is None:  # B: max|v| dx of the reference state
                            fl = float(np.max(np.abs(b["v"]))) * cfg.dx()
                        e = field_rel(a, b, f, floor=fl)
                        errs[(k, f)] = e
                        assert e <= tol[k], (k, f, e)
        out = sim.particles()
    refp = ref.particles()
    ref.close()
    return errs, out, refp


def test_c5_bench_scene_binning_bitwise_vs_reference_sort():
    cfg = block_scene(108)
    p = seed_particles(cfg, 8)
    assert len(p) == 10_077_696
    # a shuffled copy forces the full stable sort of every particle
    q = p[np.random.default_rng(0).permutation(len(p))]
    k_ref, o_ref = bind.ref_sort(cfg, q)
    with Simulation(cfg, precision=8, particles=q) as sim:
        k, o = sim.debug_sort()
    assert np.array_equal(k, k_ref)
    assert np.array_equal(o, o_ref)


def test_c5_bench_scene_state_vs_reference():
    cfg = block_scene(108)
    p = seed_particles(cfg, 8)
    _run_pair(cfg, p, 3, {1: 1e-12, 3: 1e-11})


def test_c2_two_spheres_momentum_vs_reference():
    cfg = SceneConfig.from_json(C2)
    p = seed_particles(cfg, 8)
    assert len(p) == 1_047_968
    mom = []

    def track(k, sim, ref):
        mom.append((np.asarray(sim.diagnostics().momentum, dtype=np.float64),
                    np.asarray(ref.diagnostics().momentum, dtype=np.float64)))

    m = np.sum(p["mass"].astype(np.float64))
    pscale = m * 0.05 * np.sqrt(3.0)
    g0 = np.sum(p["mass"][:, None].astype(np.float64) * p["v"], axis=0)
    _run_pair(cfg, p, 20, {1: 1e-12, 20: 1e-10}, each=track)
    gd = np.array([a for a, _ in mom])
    rd = np.array([b for _, b in mom])
    # total momentum: device vs reference at every substep, and the device's
    # drift from the initial value at the reference's level (force-free)
    assert np.max(np.abs(gd - rd)) <= 1e-12 * pscale
    drift_gpu = np.max(np.abs(gd - g0)) / pscale
    drift_ref = np.max(np.abs(rd - g0)) / pscale
    assert drift_gpu <= max(10 * drift_ref, 1e-13), (drift_gpu, drift_ref)


def test_c3_sand_column_dp_vs_reference():
    cfg = SceneConfig.from_json(C3)
    p = seed_particles(cfg, 8)
    assert len(p) == 4_194_304
    _run_pair(cfg, p, 3, {1: 1e-12, 3: 1e-11})


def test_c4_sandcastle_vs_reference():
    cfg = SceneConfig.from_json(C4)
    p = seed_particles(cfg, 8)
    assert len(p) == 10_111_224
    _run_pair(cfg, p, 3, {1: 1e-12, 3: 1e-11})


def test_twisting_bar_rotating_sticky_bc_vs_reference():
    """proj/configs/twisting_bar_ppc8.json: two sticky boxes prescribing
    v0 + omega x (x - c) with omega = (+-1, 0, 0) (grid.hpp:38-44)."""
    cfg = SceneConfig.from_json(TWIST)
    p = seed_particles(cfg, 8)
    errs, a, _ = _run_pair(cfg, p, 50, {1: 1e-12, 10: 1e-10, 50: 1e-9}, threads=1, deterministic=True,
                           floors={"x": 1.0, "v": 0.05, "F": 1.0, "B": None, "J": 1.0})
    # the bar's ends really rotate: angular velocity about x of the end slabs
    assert np.max(np.abs(a["v"][:, 1:])) > 1e-3


def test_clamp_singular_vs_reference():
    """clamp_singular (transfer.hpp:574-577): singular values of F below the
    floor are clamped after the F update.  A compressed, sheared block with a
    high floor so the clamp acts on every particle."""
    obj = {"name": "clamp", "resolution": 32, "scheme": "apic", "gravity": [0, -9.8, 0],
           "clamp_singular": True, "clamp_floor": 0.9,
           "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1e5, "nu": 0.3}],
           "bodies": [{"shape": {"kind": "box", "lo": [0.34375, 0.3125, 0.34375], "hi": [0.59375, 0.5625, 0.59375]},
                       "material": 0, "ppc": 8, "velocity": [0.2, -0.1, 0.05]}],
           "boundaries": [{"kind": "sticky", "lo": [0, 0, 0], "hi": [1, 0.25, 1]}]}
    cfg = SceneConfig.from_json(obj)
    p = seed_particles(cfg, 8)
    rng = np.random.default_rng(7)
    p["F"] = np.diag([0.8, 1.0, 0.85]) + rng.uniform(-0.02, 0.02, (len(p), 3, 3))
    errs, a, _ = _run_pair(cfg, p, 10, {1: 1e-12, 10: 1e-10}, threads=1, deterministic=True,
                           fields=("x", "v", "F", "B"))
    sv = np.linalg.svd(a["F"].astype(np.float64), compute_uv=False)
    assert np.min(sv) >= 0.9 * (1 - 1e-12)


def test_c5_bench_scene_float_vs_reference_float():
    """The bench scene in the reference's single precision (Simulation<float>,
    tools/ckmpm_main.cpp:122 `--precision single`; the bench's secondary
    figure): keys and stable order bit-exact in float, state <= 1e-5 after 2
    substeps."""
    cfg = block_scene(108)
    p = tag_volumes(seed_particles(cfg, 4))
    ref = bind.Ref(cfg, p, precision=4, threads=THREADS, deterministic=False)
    with Simulation(cfg, precision=4, particles=p) as sim:
        k, o = sim.debug_sort()
        k_ref, o_ref = bind.ref_sort(cfg, p, precision=4)
        assert np.array_equal(k, k_ref) and np.array_equal(o, o_ref)
        for _ in range(2):
            dt = ref.cfl_dt(1.0)
            assert ref.step(dt)[0] == 0
            sim.step(dt)
        a, b = sim.particles(), ref.particles()
    ref.close()
    assert np.array_equal(a["volume0"], b["volume0"])
    for f in ("x", "v", "F"):
        assert field_rel(a, b, f, floor=1.0 if f != "v" else 0.01) <= 1e-5, f


@pytest.mark.parametrize("variant", ["pic", "quadratic"])
def test_c5_bench_scene_other_transfers_vs_reference(variant):
    """The bench scene with the PIC transfer (no affine term) and with the
    quadratic B-spline baseline (27-node single grid) against the reference
    engine run the same way."""
    cfg = block_scene(108, scheme="pic") if variant == "pic" else block_scene(108, kernel="quadratic")
    p = seed_particles(cfg, 8)
    fields = ("x", "v", "F") if variant == "pic" else ("x", "v", "F", "B")
    _run_pair(cfg, p, 2, {1: 1e-12, 2: 1e-12}, fields=fields)


def test_c2_two_spheres_mls_vs_reference():
    """MLS (mls_moment / gauss_inverse4 / the force through grad Phi,
    transfer.hpp:127-150, :335-369) at 1M particles."""
    obj = dict(C2)
    obj["scheme"] = "mls"
    cfg = SceneConfig.from_json(obj)
    p = seed_particles(cfg, 8)
    _run_pair(cfg, p, 3, {1: 1e-12, 3: 1e-11})


def test_fluid_column_4m_vs_reference():
    """A J-fluid (weakly compressible, viscous: material.hpp:132-143, the
    dam-break scenes' model) column of 4,194,304 particles at res 256."""
    obj = dict(C3)
    obj["name"] = "fluid_column_4M"
    obj["materials"] = [{"model": "j_fluid", "density": 1000.0, "bulk": 10.0, "gamma": 7.15, "viscosity": 0.1}]  # configs/dam_break_reduced.json
    obj["boundaries"] = [{"kind": "slip", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]
    cfg = SceneConfig.from_json(obj)
    p = seed_particles(cfg, 8)
    assert len(p) == 4_194_304
    _run_pair(cfg, p, 3, {1: 1e-12, 3: 1e-11}, fields=("x", "v", "F", "B", "J"))
