"""ctypes mirror of include/ckmpm_b200.h (the C-ABI of the B200 transfer path).

Layouts are asserted against the C header's sizes at import of the native
library (see _lib.py).  Particle arrays are numpy structured arrays whose
layout is byte-identical to the reference's ``ckmpm::Particle<T>``
(proj/include/ckmpm/transfer.hpp:19-28): 224 B for double, 112 B for float.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

ABI_VERSION = 2

OK, ERR_CONFIG, ERR_NUMERICAL, ERR_IO, ERR_DEVICE = 0, 2, 3, 4, 5

NUM_NONE = 0
NUM_OUT_OF_DOMAIN = 1
NUM_FC_STRESS_INVERTED = 2
NUM_DP_STRESS_INVERTED = 3
NUM_FLUID_STATE_J = 4
NUM_NEAR_SINGULAR_D = 5
NUM_SINGULAR_MLS = 6
NUM_RETURN_MAP_INVERTED = 7
NUM_F_INVERTED = 8
NUM_FLUID_J = 9
NUM_NONFINITE = 10
NUM_INACTIVE_BLOCK = 11
NUM_SUBSTEP_LIMIT = 12
FLAG_QUADRATIC = 1  # ckg_config.flags: KernelKind::quadratic
FLAG_FUSED = 2  # ckg_config.flags: fused G2P2G kernel (G2P of substep n + P2G of n+1)
RECORDS_CHECKPOINT = 0
RECORDS_SNAPSHOT = 1

MAX_MATERIALS = 16
MAX_BOUNDARIES = 32

MODEL_FIXED_COROTATED, MODEL_J_FLUID, MODEL_DRUCKER_PRAGER = 0, 1, 2
MODEL_NAMES = {"fixed_corotated": 0, "j_fluid": 1, "drucker_prager": 2}
SCHEME_PIC, SCHEME_APIC, SCHEME_MLS = 0, 1, 2
SCHEME_NAMES = {"pic": 0, "apic": 1, "mls": 2}
BC_STICKY, BC_SLIP, BC_SEPARATE = 0, 1, 2
BC_NAMES = {"sticky": 0, "slip": 1, "separate": 2}

PHASE_SORT, PHASE_ACTIVATE, PHASE_CLEAR, PHASE_P2G, PHASE_GRID, PHASE_G2P = 1, 2, 3, 4, 5, 6
PHASE_NAMES = ("sort", "activate", "clear", "p2g", "grid", "g2p")

D3 = C.c_double * 3


class Material(C.Structure):
    _fields_ = [
        ("model", C.c_int32), ("_pad", C.c_int32),
        ("density", C.c_double), ("E", C.c_double), ("nu", C.c_double),
        ("mu", C.c_double), ("lambda_", C.c_double),
        ("bulk", C.c_double), ("gamma", C.c_double), ("viscosity", C.c_double),
        ("friction_angle_deg", C.c_double), ("dp_alpha", C.c_double),
    ]


class Boundary(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("_pad", C.c_int32),
        ("lo", D3), ("hi", D3), ("normal", D3), ("velocity", D3), ("omega", D3), ("center", D3),
    ]


class Config(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("precision", C.c_int32),
        ("resolution", C.c_int32), ("scheme", C.c_int32),
        ("extent", C.c_double), ("dx", C.c_double), ("inv_dx", C.c_double),
        ("gravity", D3),
        ("mass_eps", C.c_double),
        ("clamp_singular", C.c_int32), ("deterministic", C.c_int32),
        ("clamp_floor", C.c_double),
        ("n_materials", C.c_int32), ("n_boundaries", C.c_int32),
        ("materials", Material * MAX_MATERIALS),
        ("boundaries", Boundary * MAX_BOUNDARIES),
        ("device", C.c_int32), ("flags", C.c_int32),
    ]


class StepOut(C.Structure):
    _fields_ = [
        ("vmax", C.c_double),
        ("min_j", C.c_double * MAX_MATERIALS),
        ("p2g_node_visits", C.c_uint64), ("g2p_node_visits", C.c_uint64),
        ("p2g_transfers", C.c_uint64), ("g2p_transfers", C.c_uint64),
        ("phase_ms", C.c_double * 6),
        ("status", C.c_int32), ("error_code", C.c_int32),
        ("error_axis", C.c_int32), ("error_phase", C.c_int32),
        ("error_particle", C.c_uint64),
        ("active_blocks", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("sort_changed", C.c_uint64),
        ("sort_kind", C.c_int32), ("slab_migration", C.c_int32), ("substeps_done", C.c_uint64),
    ]


class FrameIn(C.Structure):
    """ckg_frame_in: the reference driver's advance_frame bookkeeping."""
    _fields_ = [
        ("time", C.c_double), ("frame_dt", C.c_double), ("frame_index", C.c_uint64),
        ("cfl", C.c_double), ("max_dt", C.c_double), ("max_substeps", C.c_uint64),
        ("vmax", C.c_double), ("min_j", C.c_double * MAX_MATERIALS),
    ]


class FrameOut(C.Structure):
    _fields_ = [
        ("substeps", C.c_uint64), ("time", C.c_double), ("last_dt", C.c_double),
        ("vmax", C.c_double), ("min_j", C.c_double * MAX_MATERIALS), ("device_ms", C.c_double),
        ("status", C.c_int32), ("error_code", C.c_int32),
        ("error_axis", C.c_int32), ("error_phase", C.c_int32),
        ("error_particle", C.c_uint64), ("active_blocks", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("graph", C.c_int32), ("_pad", C.c_int32),
        ("sort_paths", C.c_uint64 * 3),
    ]


class Diagnostics(C.Structure):
    _fields_ = [
        ("momentum", D3), ("angular", D3), ("momentum_massfree", D3),
        ("kinetic_energy", C.c_double), ("vmax", C.c_double),
    ]


def particle_dtype(precision: int) -> np.dtype:
    """numpy twin of ckmpm::Particle<T> (transfer.hpp:19-28)."""
    if precision == 8:
        return np.dtype([
            ("x", "<f8", (3,)), ("v", "<f8", (3,)), ("F", "<f8", (3, 3)), ("B", "<f8", (3, 3)),
            ("J", "<f8"), ("mass", "<f8"), ("volume0", "<f8"), ("material", "<u4"), ("_pad", "<u4"),
        ])
    if precision == 4:
        return np.dtype([
            ("x", "<f4", (3,)), ("v", "<f4", (3,)), ("F", "<f4", (3, 3)), ("B", "<f4", (3, 3)),
            ("J", "<f4"), ("mass", "<f4"), ("volume0", "<f4"), ("material", "<u4"),
        ])
    raise ValueError("precision must be 8 or 4")


assert particle_dtype(8).itemsize == 224
assert particle_dtype(4).itemsize == 112


def ptr(a: np.ndarray) -> C.c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)
