"""The C restatement (oracle/libckoracle.so) is pinned bit-exact against the
reference engine compiled unmodified (oracle/_ref/libckref.so) and against
the reference's own known-answer values (proj/tests/test_kernel.cpp:37-47,
:73-79, :130-147)."""
import ctypes as C
import os
import time

import numpy as np
import pytest

from oracle import bind
from tests.util import perturb, small_scene

from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.scene import seed_particles

HAVE_REF = os.path.exists(bind.REF_PATH)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


def test_kernel_known_answers():
    o = bind.oracle_lib()
    # test_kernel.cpp:37-47
    assert o.ckor_ck_weight_1d(0.0) == 1.0
    assert o.ckor_ck_weight_1d(1.0) == 0.0
    assert o.ckor_ck_weight_1d(-1.0) == 0.0
    assert o.ckor_ck_weight_1d(0.5) == 0.5
    assert abs(o.ckor_ck_weight_1d(0.25) - 0.9091549430918954) <= 1e-15
    assert abs(o.ckor_ck_weight_1d(0.3) - 0.8513653457281314) <= 1e-15
    assert abs(o.ckor_ck_weight_1d(0.7) - 0.14863465427186864) <= 1e-15
    # test_kernel.cpp:73-79
    assert o.ckor_ck_grad_1d(0.0) == 0.0
    assert abs(o.ckor_ck_grad_1d(0.25) + 1.0) <= 1e-15
    assert abs(o.ckor_ck_grad_1d(-0.25) - 1.0) <= 1e-15
    # axis pair (test_kernel.cpp:130-147)
    base = C.c_int32()
    v = (C.c_double * 5)()
    o.ckor_axis_pair(0.3, 1, 1.0, C.byref(base), v)
    assert base.value == 0 and abs(v[0] - 0.05) <= 1e-15
    o.ckor_axis_pair(0.3, -1, 1.0, C.byref(base), v)
    assert base.value == 0 and abs(v[0] - 0.55) <= 1e-15
    o.ckor_axis_pair(0.25, 1, 1.0, C.byref(base), v)
    assert base.value == 0 and v[0] == 0.0 and v[1] == 1.0 and v[2] == 0.0 and v[3] == 0.0 and v[4] == 0.0


@needs_ref
def test_kernel_and_math_bitwise_vs_reference():
    o, r = bind.oracle_lib(), bind.ref_lib()
    rng = np.random.default_rng(3)
    for u in rng.uniform(-1.2, 1.2, 500):
        assert o.ckor_ck_weight_1d(u) == r.ckref_ck_weight_1d(u)
        assert o.ckor_ck_grad_1d(u) == r.ckref_ck_grad_1d(u)
    b1, b2 = C.c_int32(), C.c_int32()
    v1, v2 = (C.c_double * 5)(), (C.c_double * 5)()
    for x, dx, k in zip(rng.uniform(-3, 3, 500), rng.uniform(0.01, 2, 500), rng.choice([-1, 1], 500)):
        o.ckor_axis_pair(x, int(k), dx, C.byref(b1), v1)
        r.ckref_axis_pair(x, int(k), dx, C.byref(b2), v2)
        assert b1.value == b2.value and list(v1) == list(v2)
    for s in range(300):
        F = np.eye(3) + rng.uniform(-0.4, 0.4, (3, 3))
        if s % 10 == 0:
            F[:, 2] = F[:, 1] * 1.0  # singular -> SVD fallback path
        F = np.ascontiguousarray(F)
        R1, R2 = np.zeros(9), np.zeros(9)
        o.ckor_polar_rotation(abi.ptr(F), abi.ptr(R1))
        r.ckref_polar_rotation(abi.ptr(F), abi.ptr(R2))
        assert np.array_equal(R1, R2)
        U1, S1, V1, U2, S2, V2 = (np.zeros(9), np.zeros(3), np.zeros(9), np.zeros(9), np.zeros(3), np.zeros(9))
        o.ckor_svd3(abi.ptr(F), abi.ptr(U1), abi.ptr(S1), abi.ptr(V1))
        r.ckref_svd3(abi.ptr(F), abi.ptr(U2), abi.ptr(S2), abi.ptr(V2))
        assert np.array_equal(U1, U2) and np.array_equal(S1, S2) and np.array_equal(V1, V2)


def _bitwise_equal(a, b):
    return a.tobytes() == b.tobytes()


CASES = [
    dict(scheme="pic", model="fixed_corotated", bc="sticky"),
    dict(scheme="apic", model="fixed_corotated", bc="sticky"),
    dict(scheme="mls", model="fixed_corotated", bc="none"),
    dict(scheme="apic", model="drucker_prager", bc="separate"),
    dict(scheme="apic", model="j_fluid", bc="slip"),
    dict(scheme="pic", model="j_fluid", bc="separate"),
]


@needs_ref
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['scheme']}-{c['model']}-{c['bc']}")
def test_oracle_steps_bitwise_vs_reference(case):
    cfg = small_scene(res=32, lo=(0.375, 0.3125, 0.375), hi=(0.5, 0.4375, 0.5), **case)
    p0 = perturb(seed_particles(cfg), seed=7, fscale=0.02)
    ref = bind.Ref(cfg, p0, threads=1, deterministic=True)
    orc = bind.Oracle(cfg, p0)
    for step in range(4):
        dt = ref.cfl_dt(1.0)
        assert dt == orc.cfl_dt(1.0)
        rc1, m1 = ref.step(dt)
        rc2, m2, out = orc.step(dt)
        assert rc1 == rc2 and m1 == m2, (m1, m2)
        assert _bitwise_equal(ref.particles(), orc.particles()), f"step {step}"
        c1, n1 = ref.grid()
        c2, n2 = orc.grid()
        assert np.array_equal(c1, c2) and np.array_equal(n1, n2)
    d1, d2 = ref.diagnostics(), orc.diagnostics()
    assert bytes(d1) == bytes(d2)


@needs_ref
def test_oracle_sort_matches_reference():
    cfg = small_scene(res=40, lo=(0.3, 0.3, 0.3), hi=(0.55, 0.5, 0.6))
    p = perturb(seed_particles(cfg), seed=2, xscale=2.0, dx=1.0 / 40)
    rng = np.random.default_rng(0)
    p = p[rng.permutation(len(p))]
    k1, o1 = bind.ref_sort(cfg, p)
    orc = bind.Oracle(cfg, p)
    k2, o2 = orc.sort()
    assert np.array_equal(k1, k2) and np.array_equal(o1, o2)


@needs_ref
def test_oracle_errors_match_reference():
    cfg = small_scene(res=32)
    p = seed_particles(cfg)
    p["x"][5, 0] = 1.5 / 32  # violates the 2-cell inset on axis 0
    ref = bind.Ref(cfg, p)
    orc = bind.Oracle(cfg, p)
    rc1, m1 = ref.step(1e-4)
    rc2, m2, out = orc.step(1e-4)
    assert rc1 == rc2 == 3 and m1 == m2
    assert "violates the 2-cell domain inset on axis 0" in m1


@needs_ref
def test_reference_pool_resize_between_instances():
    """Alternating thread counts across reference instances in one process
    (the at-size GPU tests do): the shim's prepare_pool absorbs the
    reference pool's spurious wake-ups after a resize, which otherwise
    surface as std::bad_function_call from the next parallel loop."""
    cfg = small_scene(res=32, lo=(0.375, 0.3125, 0.375), hi=(0.5, 0.4375, 0.5))
    p0 = seed_particles(cfg)
    for threads in (4, 2, 4, 1, 3):
        ref = bind.Ref(cfg, p0, threads=threads, deterministic=False)
        time.sleep(0.05)  # let freshly started workers run first
        for _ in range(2):
            rc, msg = ref.step(ref.cfl_dt(1.0))
            assert rc == 0, msg
        ref.close()
