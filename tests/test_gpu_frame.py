"""Device frame driver (ckg_advance_frame): advance_frame
(simulation.hpp:193-211) as one CUDA-graph launch with the step size, the
frame-boundary test and the sort path decided on the GPU.  Checked against the
host loop over ckg_step (same library, host cfl_dt) and against the reference
engine's own advance_frame loop (oracle/_ref)."""
import numpy as np
import pytest

from oracle import bind
from paper_2412_10399_b200.scene import NumericalError, OutOfDomainError, SceneConfig, seed_particles
from tests.gpu_util import field_rel, gpu_sim, match_by_tag, tag_volumes
from tests.util import small_scene

pytestmark = pytest.mark.gpu


def _ref_advance_frame(ref, cfg, book):
    """The reference's advance_frame loop (simulation.hpp:193-211) over its
    own cfl_dt and step, with the same T arithmetic for time_."""
    T = np.float64
    frame_dt = T(cfg.frame_dt)
    frame_end = frame_dt * T(book["frame"] + 1)
    steps = 0
    while True:
        rem = frame_end - T(book["time"])
        if rem <= frame_dt * T(1e-9):
            book["time"] = float(frame_end)
            break
        dt = ref.cfl_dt(float(rem))
        rc, msg = ref.step(dt)
        assert rc == 0, msg
        book["time"] = float(T(book["time"]) + T(dt))
        steps += 1
    book["frame"] += 1
    return steps


def _pair(cfg, p):
    """(device frame driver, host loop): the CUDA-graph frame driver runs the
    separate P2G / G2P kernels; the host loop runs fused G2P2G substeps, so
    the two paths are checked against each other as well."""
    return gpu_sim(cfg, p), gpu_sim(cfg, p, fused=True)


def _compare_states(a, b, tol):
    a, b = match_by_tag(a, b)
    for f, fl in (("x", 1.0), ("v", 0.1), ("F", 1.0), ("B", 1e-4), ("J", 1.0)):
        assert field_rel(a, b, f, fl) <= tol, f


def test_frame_device_matches_host_loop_and_reference():
    cfg = small_scene(res=32, bc="sticky")
    p = tag_volumes(seed_particles(cfg))
    dev, host = _pair(cfg, p)
    ref = bind.Ref(cfg, p)
    book = {"time": 0.0, "frame": 0}
    for frame in range(3):
        n_dev = dev.advance_frame()
        n_host = host.advance_frame(device=False)
        n_ref = _ref_advance_frame(ref, cfg, book)
        assert n_dev == n_host == n_ref > 4
        assert dev.last_frame.graph == 1
        assert dev.time() == host.time() == book["time"]
        assert dev.step_count() == host.step_count()
        assert dev.frame_index() == host.frame_index() == frame + 1
        # the device loop's vmax_ feeds the next frame's first dt exactly
        assert dev.cfl_dt(1.0) == host.cfl_dt(1.0)
    _compare_states(dev.particles(), host.particles(), 1e-10)
    _compare_states(dev.particles(), ref.particles(), 1e-8)
    assert dev.counters().g2p_transfers == host.counters().g2p_transfers


@pytest.mark.parametrize("velocity,path", [((7.5, 0.0, 0.0), 1), ((15.0, 15.0, 15.0), 2)],
                         ids=["padded_radix", "full_radix"])
def test_frame_sort_paths(velocity, path):
    """More block crossers per substep than the one-CTA crosser sort takes
    (> 8192): up to n/8 of them go through the fixed-size padded radix sort,
    more through the full radix sort -- the graph's IF nodes pick the path on
    the device; results match the host loop's incremental / full sort."""
    obj = {"resolution": 128, "scheme": "apic", "gravity": [0, 0, 0], "frame_dt": 1.0 / 240,
           "materials": [{"model": "fixed_corotated", "density": 1000.0, "E": 1e5, "nu": 0.4}],
           "bodies": [{"shape": {"kind": "box", "lo": [0.25, 0.25, 0.25], "hi": [0.5, 0.5, 0.5]},
                       "material": 0, "ppc": 8, "velocity": list(velocity)}],
           "boundaries": []}
    cfg = SceneConfig.from_json(obj)
    p = tag_volumes(seed_particles(cfg))
    assert len(p) > 8 * 8192
    dev, host = _pair(cfg, p)
    n_dev = dev.advance_frame()
    n_host = host.advance_frame(device=False)
    assert n_dev == n_host > 4
    assert dev.time() == host.time()
    assert dev.last_frame.sort_paths[path] > 0, list(dev.last_frame.sort_paths)
    _compare_states(dev.particles(), host.particles(), 1e-10)


def test_frame_fluid_matches_host_loop():
    cfg = small_scene(model="j_fluid", res=32, bc="slip", gravity=(0, -9.8, 0))
    p = tag_volumes(seed_particles(cfg))
    dev, host = _pair(cfg, p)
    for _ in range(2):
        n_dev = dev.advance_frame()
        n_host = host.advance_frame(device=False)
        assert n_dev == n_host
        # std::pow on the host vs CUDA pow for the fluid sound speed: the dt
        # sequences agree to an ulp
        assert abs(dev.time() - host.time()) <= 1e-15
    _compare_states(dev.particles(), host.particles(), 1e-9)


def test_frame_substep_limit():
    cfg = small_scene(res=32)
    cfg.max_substeps_per_frame = 3
    p = seed_particles(cfg)
    dev, host = _pair(cfg, p)
    with pytest.raises(NumericalError) as e_dev:
        dev.advance_frame()
    with pytest.raises(NumericalError) as e_host:
        host.advance_frame(device=False)
    assert str(e_dev.value) == str(e_host.value)
    assert "substep limit exceeded within one frame at t = " in str(e_dev.value)
    assert dev.step_count() == host.step_count() == 4
    assert dev.time() == host.time()
    assert dev.frame_index() == host.frame_index() == 0


def test_frame_error_mid_frame():
    """A body leaving the domain inset during the frame: the same exception,
    particle index and bookkeeping as the host loop."""
    cfg = small_scene(res=32, bc="none", gravity=(0, 0, 0), velocity=(12.0, 0.0, 0.0),
                      lo=(0.6, 0.4, 0.4), hi=(0.8, 0.6, 0.6))
    cfg.frame_dt = 1.0 / 30
    p = seed_particles(cfg)
    dev, host = _pair(cfg, p)
    with pytest.raises(OutOfDomainError) as e_dev:
        dev.advance_frame()
    with pytest.raises(OutOfDomainError) as e_host:
        host.advance_frame(device=False)
    assert str(e_dev.value) == str(e_host.value)
    assert e_dev.value.particle_index == e_host.value.particle_index
    assert dev.step_count() == host.step_count() > 1
    assert dev.time() == host.time()
    _compare_states(dev.particles(), host.particles(), 1e-10)
