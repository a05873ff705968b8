"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the two CPU checkers.

* ``Ref``  -> oracle/_ref/libckref.so : the reference engine itself
  (/root/reference/proj/include/ckmpm, compiled unmodified by oracle/Makefile).
* ``Oracle`` -> oracle/libckoracle.so : the plain-C restatement
  (oracle/ckmpm_oracle.c), pinned bit-exact against ``Ref``.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2412_10399_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libckref.so")
ORACLE_PATH = os.path.join(HERE, "libckoracle.so")


class Body(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("axis", C.c_int32), ("center", C.c_double * 3),
        ("radius", C.c_double), ("inner_radius", C.c_double), ("half_length", C.c_double),
        ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("material", C.c_uint32), ("ppc", C.c_int32),
        ("seed", C.c_uint64), ("velocity", C.c_double * 3), ("shear_slope", C.c_double),
        ("omega", C.c_double * 3),
    ]


class Extra(C.Structure):
    _fields_ = [("cfl", C.c_double), ("frame_dt", C.c_double), ("max_dt", C.c_double),
                ("threads", C.c_int32), ("_pad", C.c_int32)]


_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(f"{REF_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        l = C.CDLL(REF_PATH)
        vp, P = C.c_void_p, C.POINTER
        l.ckref_finalize_material.argtypes = [P(abi.Material), C.c_int32, C.c_char_p, C.c_int32]
        l.ckref_seed.argtypes = [P(abi.Config), P(Body), C.c_int32, vp, C.c_int64]
        l.ckref_seed.restype = C.c_int64
        l.ckref_sim_create.argtypes = [P(abi.Config), P(Extra), vp, C.c_uint64, C.c_char_p, C.c_int32]
        l.ckref_sim_create.restype = vp
        l.ckref_sim_destroy.argtypes = [vp]
        l.ckref_sim_step.argtypes = [vp, C.c_double, C.c_char_p, C.c_int32]
        l.ckref_sim_cfl_dt.argtypes = [vp, C.c_double]
        l.ckref_sim_cfl_dt.restype = C.c_double
        l.ckref_sim_count.argtypes = [vp]
        l.ckref_sim_count.restype = C.c_uint64
        l.ckref_sim_particles.argtypes = [vp, vp, C.c_uint64]
        l.ckref_sim_timers.argtypes = [vp, P(C.c_double)]
        l.ckref_sim_active_blocks.argtypes = [vp]
        l.ckref_sim_active_blocks.restype = C.c_uint64
        l.ckref_sim_grid.argtypes = [vp, vp, vp, C.c_uint64]
        l.ckref_sim_diagnostics.argtypes = [vp, P(abi.Diagnostics)]
        l.ckref_sim_write_checkpoint.argtypes = [vp, C.c_char_p]
        l.ckref_sim_write_checkpoint.restype = C.c_int32
        l.ckref_sim_write_snapshot.argtypes = [vp, C.c_char_p, C.c_int32, C.c_int32]
        l.ckref_sim_write_snapshot.restype = C.c_int32
        l.ckref_sim_mass_epsilon.argtypes = [vp]
        l.ckref_sim_mass_epsilon.restype = C.c_double
        l.ckref_p2g.argtypes = [P(abi.Config), vp, C.c_uint64, C.c_double, vp, vp, C.c_uint64, C.c_char_p, C.c_int32]
        l.ckref_p2g.restype = C.c_int64
        l.ckref_sort.argtypes = [P(abi.Config), vp, C.c_uint64, vp, vp]
        l.ckref_ck_weight_1d.argtypes = [C.c_double]
        l.ckref_ck_weight_1d.restype = C.c_double
        l.ckref_ck_grad_1d.argtypes = [C.c_double]
        l.ckref_ck_grad_1d.restype = C.c_double
        l.ckref_axis_pair.argtypes = [C.c_double, C.c_int32, C.c_double, P(C.c_int32), P(C.c_double)]
        l.ckref_polar_rotation.argtypes = [vp, vp]
        l.ckref_svd3.argtypes = [vp, vp, vp, vp]
        l.ckref_return_map_dp.argtypes = [vp, C.c_double, C.c_double, C.c_double, vp]
        _ref = l
    return _ref


def oracle_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_PATH):
            raise FileNotFoundError(f"{ORACLE_PATH} missing: run `make -C oracle`")
        l = C.CDLL(ORACLE_PATH)
        vp, P = C.c_void_p, C.POINTER
        l.ckor_create.argtypes = [P(abi.Config), vp, C.c_uint64]
        l.ckor_create.restype = vp
        l.ckor_destroy.argtypes = [vp]
        l.ckor_step.argtypes = [vp, C.c_double, P(abi.StepOut), C.c_char_p, C.c_int32]
        l.ckor_step_phases.argtypes = [vp, C.c_double, C.c_int32, P(abi.StepOut), C.c_char_p, C.c_int32]
        l.ckor_count.argtypes = [vp]
        l.ckor_count.restype = C.c_uint64
        l.ckor_particles.argtypes = [vp, vp]
        l.ckor_cfl_dt.argtypes = [vp, C.c_double, C.c_double, C.c_double]
        l.ckor_cfl_dt.restype = C.c_double
        l.ckor_vmax.argtypes = [vp]
        l.ckor_vmax.restype = C.c_double
        l.ckor_active_blocks.argtypes = [vp]
        l.ckor_active_blocks.restype = C.c_uint64
        l.ckor_grid.argtypes = [vp, vp, vp, C.c_uint64]
        l.ckor_sort.argtypes = [vp, vp, vp]
        l.ckor_diagnostics.argtypes = [vp, P(abi.Diagnostics)]
        l.ckor_ck_weight_1d.argtypes = [C.c_double]
        l.ckor_ck_weight_1d.restype = C.c_double
        l.ckor_ck_grad_1d.argtypes = [C.c_double]
        l.ckor_ck_grad_1d.restype = C.c_double
        l.ckor_axis_pair.argtypes = [C.c_double, C.c_int32, C.c_double, P(C.c_int32), P(C.c_double)]
        l.ckor_polar_rotation.argtypes = [vp, vp]
        l.ckor_svd3.argtypes = [vp, vp, vp, vp]
        _orc = l
    return _orc


def bodies_from_scene(cfg):
    kinds = {"sphere": 0, "box": 1, "cylinder": 2}
    arr = (Body * max(1, len(cfg.bodies)))()
    for i, b in enumerate(cfg.bodies):
        d = arr[i]
        s = b.shape
        d.kind, d.axis = kinds[s.kind], s.axis
        d.radius, d.inner_radius, d.half_length = s.radius, s.inner_radius, s.half_length
        for a in range(3):
            d.center[a], d.lo[a], d.hi[a] = s.center[a], s.lo[a], s.hi[a]
            d.velocity[a], d.omega[a] = b.velocity[a], b.omega[a]
        d.material, d.ppc, d.seed, d.shear_slope = b.material, b.ppc, b.seed, b.shear_slope
    return arr


def ref_seed(cfg, precision=8):
    abic = _cfg(cfg, precision)
    bodies = bodies_from_scene(cfg)
    n = ref_lib().ckref_seed(C.byref(abic), bodies, len(cfg.bodies), None, 0)
    out = np.zeros(n, dtype=abi.particle_dtype(precision))
    ref_lib().ckref_seed(C.byref(abic), bodies, len(cfg.bodies), abi.ptr(out), n)
    return out


def _cfg(cfg, precision, mass_eps=0.0):
    from paper_2412_10399_b200.scene import to_abi_config
    return to_abi_config(cfg, precision, mass_eps)


class Ref:
    """The reference Simulation<T> (compiled reference headers)."""

    def __init__(self, cfg, particles, precision=8, mass_eps=None, threads=1, deterministic=True):
        from paper_2412_10399_b200.scene import mass_epsilon
        self.precision = precision
        me = mass_epsilon(particles, precision) if mass_eps is None else mass_eps
        self.cfgabi = _cfg(cfg, precision, me)
        self.cfgabi.deterministic = int(deterministic)
        self.extra = Extra(cfg.cfl, cfg.frame_dt, cfg.max_dt, threads, 0)
        p = np.ascontiguousarray(particles)
        err = C.create_string_buffer(512)
        self.h = ref_lib().ckref_sim_create(C.byref(self.cfgabi), C.byref(self.extra), abi.ptr(p), len(p), err, 512)
        if not self.h:
            raise RuntimeError("ckref_sim_create: " + err.value.decode())
        self.n = len(p)

    def step(self, dt):
        err = C.create_string_buffer(512)
        rc = ref_lib().ckref_sim_step(self.h, float(dt), err, 512)
        return rc, err.value.decode()

    def cfl_dt(self, remaining):
        return ref_lib().ckref_sim_cfl_dt(self.h, float(remaining))

    def particles(self):
        out = np.zeros(self.n, dtype=abi.particle_dtype(self.precision))
        ref_lib().ckref_sim_particles(self.h, abi.ptr(out), self.n)
        return out

    def grid(self):
        nb = ref_lib().ckref_sim_active_blocks(self.h)
        coords = np.zeros((nb, 3), dtype=np.int32)
        nodes = np.zeros((nb, 128, 4), dtype=np.float64)
        ref_lib().ckref_sim_grid(self.h, abi.ptr(coords), abi.ptr(nodes), nb)
        return coords, nodes

    def active_blocks(self):
        return int(ref_lib().ckref_sim_active_blocks(self.h))

    def timers(self):
        t = (C.c_double * 6)()
        ref_lib().ckref_sim_timers(self.h, t)
        return list(t)

    def diagnostics(self):
        d = abi.Diagnostics()
        ref_lib().ckref_sim_diagnostics(self.h, C.byref(d))
        return d

    def write_checkpoint(self, path):
        return ref_lib().ckref_sim_write_checkpoint(self.h, str(path).encode())

    def write_snapshot(self, path, frame, binary=True):
        return ref_lib().ckref_sim_write_snapshot(self.h, str(path).encode(), int(frame), int(binary))

    def close(self):
        if self.h:
            ref_lib().ckref_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_p2g(cfg, particles, dt, precision=8, mass_eps=None):
    from paper_2412_10399_b200.scene import mass_epsilon
    me = mass_epsilon(particles, precision) if mass_eps is None else mass_eps
    c = _cfg(cfg, precision, me)
    p = np.ascontiguousarray(particles)
    err = C.create_string_buffer(512)
    nb = ref_lib().ckref_p2g(C.byref(c), abi.ptr(p), len(p), float(dt), None, None, 0, err, 512)
    if nb < 0:
        return int(-nb), err.value.decode(), None, None
    coords = np.zeros((nb, 3), dtype=np.int32)
    nodes = np.zeros((nb, 128, 4), dtype=np.float64)
    ref_lib().ckref_p2g(C.byref(c), abi.ptr(p), len(p), float(dt), abi.ptr(coords), abi.ptr(nodes), nb, err, 512)
    return 0, "", coords, nodes


def ref_sort(cfg, particles, precision=8):
    c = _cfg(cfg, precision)
    p = np.ascontiguousarray(particles)
    keys = np.zeros(len(p), dtype=np.uint32)
    order = np.zeros(len(p), dtype=np.uint32)
    ref_lib().ckref_sort(C.byref(c), abi.ptr(p), len(p), abi.ptr(keys), abi.ptr(order))
    return keys, order


class Oracle:
    """The plain-C restatement (double only)."""

    def __init__(self, cfg, particles, mass_eps=None):
        from paper_2412_10399_b200.scene import mass_epsilon
        me = mass_epsilon(particles, 8) if mass_eps is None else mass_eps
        self.cfg = cfg
        self.cfgabi = _cfg(cfg, 8, me)
        p = np.ascontiguousarray(particles)
        self.h = oracle_lib().ckor_create(C.byref(self.cfgabi), abi.ptr(p), len(p))
        self.n = len(p)

    def step(self, dt, stop_after=abi.PHASE_G2P):
        out = abi.StepOut()
        err = C.create_string_buffer(512)
        rc = oracle_lib().ckor_step_phases(self.h, float(dt), int(stop_after), C.byref(out), err, 512)
        return rc, err.value.decode(), out

    def cfl_dt(self, remaining):
        return oracle_lib().ckor_cfl_dt(self.h, self.cfg.cfl, self.cfg.max_dt, float(remaining))

    def particles(self):
        out = np.zeros(self.n, dtype=abi.particle_dtype(8))
        oracle_lib().ckor_particles(self.h, abi.ptr(out))
        return out

    def grid(self):
        nb = oracle_lib().ckor_active_blocks(self.h)
        coords = np.zeros((nb, 3), dtype=np.int32)
        nodes = np.zeros((nb, 128, 4), dtype=np.float64)
        oracle_lib().ckor_grid(self.h, abi.ptr(coords), abi.ptr(nodes), nb)
        return coords, nodes

    def sort(self):
        keys = np.zeros(self.n, dtype=np.uint32)
        order = np.zeros(self.n, dtype=np.uint32)
        oracle_lib().ckor_sort(self.h, abi.ptr(keys), abi.ptr(order))
        return keys, order

    def diagnostics(self):
        d = abi.Diagnostics()
        oracle_lib().ckor_diagnostics(self.h, C.byref(d))
        return d

    def close(self):
        if self.h:
            oracle_lib().ckor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
