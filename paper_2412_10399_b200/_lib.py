"""Loader for the in-tree native library libckmpm_b200.so (sm_100a).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of any compute entry point raises.  Build it with ``make`` or
``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CKMPM_B200_LIB") or os.path.join(_HERE, "libckmpm_b200.so")

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def _declare(lib: C.CDLL) -> None:
    P = C.POINTER
    vp = C.c_void_p
    u64 = C.c_uint64
    i32 = C.c_int32
    lib.ckg_abi_version.restype = i32
    lib.ckg_build_info.restype = C.c_char_p
    lib.ckg_status_string.argtypes = [i32]
    lib.ckg_status_string.restype = C.c_char_p
    lib.ckg_create.argtypes = [P(abi.Config), P(vp)]
    lib.ckg_create.restype = i32
    lib.ckg_destroy.argtypes = [vp]
    lib.ckg_destroy.restype = None
    lib.ckg_upload.argtypes = [vp, vp, u64]
    lib.ckg_upload.restype = i32
    lib.ckg_download.argtypes = [vp, vp, u64]
    lib.ckg_download.restype = i32
    lib.ckg_particle_count.argtypes = [vp]
    lib.ckg_particle_count.restype = u64
    lib.ckg_fused.argtypes = [vp]
    lib.ckg_fused.restype = i32
    lib.ckg_set_mass_epsilon.argtypes = [vp, C.c_double]
    lib.ckg_set_mass_epsilon.restype = i32
    lib.ckg_step.argtypes = [vp, C.c_double, P(abi.StepOut)]
    lib.ckg_step.restype = i32
    lib.ckg_step_many.argtypes = [vp, C.c_double, i32, P(abi.StepOut)]
    lib.ckg_step_many.restype = i32
    lib.ckg_record_bytes.argtypes = [vp, i32]
    lib.ckg_record_bytes.restype = u64
    lib.ckg_pack_records.argtypes = [vp, i32, vp, u64, i32]
    lib.ckg_pack_records.restype = i32
    lib.ckg_records_wait.argtypes = [vp]
    lib.ckg_records_wait.restype = i32
    lib.ckg_advance_frame.argtypes = [vp, P(abi.FrameIn), P(abi.FrameOut)]
    lib.ckg_advance_frame.restype = i32
    lib.ckg_step_phases.argtypes = [vp, C.c_double, i32, P(abi.StepOut)]
    lib.ckg_step_phases.restype = i32
    lib.ckg_debug_sort.argtypes = [vp, vp, vp, u64]
    lib.ckg_debug_sort.restype = i32
    lib.ckg_debug_bases.argtypes = [vp, vp, u64]
    lib.ckg_debug_bases.restype = i32
    lib.ckg_grid_active_block_count.argtypes = [vp]
    lib.ckg_grid_active_block_count.restype = u64
    lib.ckg_grid_download.argtypes = [vp, vp, vp, u64]
    lib.ckg_grid_download.restype = i32
    lib.ckg_grid_totals.argtypes = [vp, P(C.c_double), P(C.c_double)]
    lib.ckg_grid_totals.restype = i32
    lib.ckg_diagnostics_compute.argtypes = [vp, P(abi.Diagnostics)]
    lib.ckg_diagnostics_compute.restype = i32
    lib.ckg_timer_mark.argtypes = [vp, i32]
    lib.ckg_timer_mark.restype = i32
    lib.ckg_timer_elapsed.argtypes = [vp, i32, i32, P(C.c_double)]
    lib.ckg_timer_elapsed.restype = i32
    lib.ckg_slab_set.argtypes = [vp, i32, i32, i32, i32]
    lib.ckg_slab_set.restype = i32
    lib.ckg_slab_bin.argtypes = [vp, C.c_double, vp]
    lib.ckg_slab_bin.restype = i32
    lib.ckg_slab_p2g.argtypes = [vp, vp, P(u64)]
    lib.ckg_slab_p2g.restype = i32
    lib.ckg_slab_p2g_part.argtypes = [vp, vp, P(u64), i32]
    lib.ckg_slab_p2g_part.restype = i32
    lib.ckg_slab_halo.argtypes = [vp, i32, i32, vp]
    lib.ckg_slab_halo.restype = i32
    lib.ckg_slab_grid.argtypes = [vp]
    lib.ckg_slab_grid.restype = i32
    lib.ckg_slab_g2p.argtypes = [vp, P(u64)]
    lib.ckg_slab_g2p.restype = i32
    lib.ckg_slab_pack.argtypes = [vp, u64, vp, vp]
    lib.ckg_slab_pack.restype = i32
    lib.ckg_slab_finish.argtypes = [vp, vp, u64, vp, u64, P(abi.StepOut)]
    lib.ckg_slab_finish.restype = i32
    lib.ckg_slab_record_words.restype = i32
    lib.ckg_slab_tile_words.restype = i32
    lib.ckg_slab_plane_counts.argtypes = [vp, P(u64)]
    lib.ckg_slab_plane_counts.restype = i32
    lib.ckg_slab_rebound.argtypes = [vp, i32, i32]
    lib.ckg_slab_rebound.restype = i32
    lib.ckg_stream.argtypes = [vp]
    lib.ckg_stream.restype = vp
    lib.ckg_last_error_message.argtypes = [vp, C.c_char_p, u64]
    lib.ckg_last_error_message.restype = i32


EXPORTED = (
    "ckg_abi_version", "ckg_build_info", "ckg_status_string", "ckg_create", "ckg_destroy",
    "ckg_upload", "ckg_download", "ckg_particle_count", "ckg_fused", "ckg_set_mass_epsilon", "ckg_step",
    "ckg_step_many", "ckg_step_phases", "ckg_advance_frame", "ckg_record_bytes", "ckg_pack_records",
    "ckg_records_wait", "ckg_debug_sort", "ckg_debug_bases",
    "ckg_grid_active_block_count", "ckg_grid_download", "ckg_grid_totals",
    "ckg_diagnostics_compute", "ckg_timer_mark", "ckg_timer_elapsed", "ckg_last_error_message",
    "ckg_slab_set", "ckg_slab_bin", "ckg_slab_p2g", "ckg_slab_p2g_part", "ckg_slab_halo", "ckg_slab_grid", "ckg_slab_g2p",
    "ckg_slab_pack", "ckg_slab_finish", "ckg_slab_record_words", "ckg_slab_tile_words", "ckg_stream", "ckg_slab_plane_counts", "ckg_slab_rebound",
)


def lib() -> C.CDLL:
    """The loaded native library (raises NativeLibraryMissing if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `make` (no CPU fallback exists by design)")
        l = C.CDLL(LIB_PATH)
        _declare(l)
        if l.ckg_abi_version() != abi.ABI_VERSION:
            raise NativeLibraryMissing("libckmpm_b200.so ABI version mismatch; rebuild")
        _lib = l
    return _lib
