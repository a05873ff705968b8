"""Python mirror of ``ckmpm::Simulation<T>`` over the B200 C-ABI.

Same public surface and error behaviour as the reference driver
(proj/include/ckmpm/simulation.hpp:85-219): ``step``, ``advance_frame``,
``cfl_dt``, ``particles``, ``restore``, ``diagnostics``, ``grid()`` facade,
``timers``/``counters``, ``mass_epsilon``, ``time``, ``step_count``,
``frame_index``.  The substep itself runs entirely on the GPU
(libckmpm_b200.so); this class only holds the host-side bookkeeping the
reference keeps on the host (time, frame schedule, CFL from vmax/minJ).

The C++ drop-in for native callers is include/ckmpm_b200/simulation.hpp;
this module is what tests and bench.py drive.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import abi
from ._lib import lib
from .scene import (ConfigError, DeviceError, InvertedElementError, IoError, NumericalError,
                    OutOfDomainError, SceneConfig, mass_epsilon, seed_particles, to_abi_config)

_INVERTED = {abi.NUM_FC_STRESS_INVERTED, abi.NUM_DP_STRESS_INVERTED, abi.NUM_RETURN_MAP_INVERTED,
             abi.NUM_F_INVERTED}


@dataclass
class PhaseTimers:
    """PhaseTimers (simulation.hpp:34-42), seconds of device time."""
    sort_s: float = 0.0
    activate_s: float = 0.0
    clear_s: float = 0.0
    p2g_s: float = 0.0
    grid_s: float = 0.0
    g2p_s: float = 0.0
    substeps: int = 0

    def total(self) -> float:
        return self.sort_s + self.activate_s + self.clear_s + self.p2g_s + self.grid_s + self.g2p_s

    def transfer_total(self) -> float:
        return self.p2g_s + self.g2p_s


@dataclass
class TransferCounters:
    """TransferCounters (transfer.hpp:32-45)."""
    p2g_node_visits: int = 0
    g2p_node_visits: int = 0
    p2g_transfers: int = 0
    g2p_transfers: int = 0


@dataclass
class DiagnosticsRow:
    """DiagnosticsRow<T> (simulation.hpp:44-53)."""
    step: int
    time: float
    momentum: np.ndarray
    angular: np.ndarray
    momentum_massfree: np.ndarray
    kinetic_energy: float
    vmax: float


def _raise_for(ctx, rc: int, out: Optional[abi.StepOut] = None):
    if rc == abi.OK:
        return
    buf = C.create_string_buffer(512)
    lib().ckg_last_error_message(ctx, buf, 512)
    msg = buf.value.decode()
    if rc == abi.ERR_CONFIG:
        raise ConfigError(msg or "invalid argument")
    if rc == abi.ERR_NUMERICAL:
        code = out.error_code if out is not None else 0
        if code == abi.NUM_OUT_OF_DOMAIN:
            raise OutOfDomainError(int(out.error_particle), msg)
        if code in _INVERTED:
            raise InvertedElementError(msg)
        raise NumericalError(msg)
    raise DeviceError(msg or f"device error {rc}")


class GridFacade:
    """BlockSparseGrid<T> read-side facade over the device grid (grid.hpp:75-281)."""

    def __init__(self, sim: "Simulation"):
        self._sim = sim

    def active_block_count(self) -> int:
        return int(lib().ckg_grid_active_block_count(self._sim._ctx))

    def blocks(self):
        """(coords (nb,3) int32, nodes (nb,128,4) float64) in directory order."""
        nb = self.active_block_count()
        coords = np.zeros((nb, 3), dtype=np.int32)
        nodes = np.zeros((nb, 128, 4), dtype=np.float64)
        rc = lib().ckg_grid_download(self._sim._ctx, abi.ptr(coords), abi.ptr(nodes), nb)
        _raise_for(self._sim._ctx, rc)
        return coords, nodes

    def total_mass(self, slot: int) -> float:
        m = (C.c_double * 2)()
        p = (C.c_double * 6)()
        _raise_for(self._sim._ctx, lib().ckg_grid_totals(self._sim._ctx, m, p))
        return float(m[slot])

    def total_momentum(self, slot: int) -> np.ndarray:
        m = (C.c_double * 2)()
        p = (C.c_double * 6)()
        _raise_for(self._sim._ctx, lib().ckg_grid_totals(self._sim._ctx, m, p))
        return np.array(p[slot * 3: slot * 3 + 3])

    def dx(self) -> float:
        return float(self._sim._abi_cfg.dx)


class Simulation:
    """B200 twin of ckmpm::Simulation<T> (precision 8 = double, 4 = float)."""

    def __init__(self, cfg: SceneConfig, precision: int = 8, device: int = 0,
                 particles: Optional[np.ndarray] = None, fused: Optional[bool] = None):
        """fused: True = the fused G2P2G kernel where supported
        (CKG_FLAG_FUSED); None/False = the library default (separate P2G /
        G2P kernels unless CKMPM_FUSED=1)."""
        cfg.validate()
        self.cfg = cfg
        self.precision = precision
        self._T = np.float64 if precision == 8 else np.float32
        host = seed_particles(cfg, precision) if particles is None else np.ascontiguousarray(particles)
        self._mass_eps = mass_epsilon(host, precision)
        self._abi_cfg = to_abi_config(cfg, precision, self._mass_eps, device)
        if fused:
            self._abi_cfg.flags |= abi.FLAG_FUSED
        ctx = C.c_void_p()
        rc = lib().ckg_create(C.byref(self._abi_cfg), C.byref(ctx))
        if rc != abi.OK:
            raise (ConfigError if rc == abi.ERR_CONFIG else DeviceError)(f"ckg_create failed ({rc})")
        self._ctx = ctx
        self._n = len(host)
        self._time = 0.0
        self._step_count = 0
        self._frame_index = 0
        self._timers = PhaseTimers()
        self._counters = TransferCounters()
        self._upload(host)
        self._refresh_velocity_stats(host)

    # -- lifetime -------------------------------------------------------
    def close(self):
        if getattr(self, "_ctx", None):
            lib().ckg_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- state ----------------------------------------------------------
    def _upload(self, host: np.ndarray):
        host = np.ascontiguousarray(host, dtype=abi.particle_dtype(self.precision))
        _raise_for(self._ctx, lib().ckg_upload(self._ctx, abi.ptr(host), len(host)))
        self._n = len(host)

    def _refresh_velocity_stats(self, host: np.ndarray):
        """refresh_velocity_stats (simulation.hpp:234-243)."""
        v = host["v"].astype(self._T)
        s = np.sqrt((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2]) if len(v) else np.zeros(1)
        self._vmax = float(np.max(s)) if len(s) else 0.0
        self._min_j = [1.0] * len(self.cfg.materials)
        for mi, m in enumerate(self.cfg.materials):
            if m.is_fluid:
                sel = host["J"][host["material"] == mi]
                if len(sel):
                    self._min_j[mi] = min(1.0, float(np.min(sel)))

    def particles(self) -> np.ndarray:
        """Current particle state in the device's (sorted) order, Particle<T> layout."""
        out = np.zeros(self._n, dtype=abi.particle_dtype(self.precision))
        _raise_for(self._ctx, lib().ckg_download(self._ctx, abi.ptr(out), self._n))
        return out

    def set_particles(self, host: np.ndarray):
        """Write-through of the non-const particles() accessor (simulation.hpp:106)."""
        self._upload(host)

    def restore(self, particles: np.ndarray, time: float, step: int, frame: int, mass_eps: float):
        """Simulation::restore (simulation.hpp:120-129)."""
        self._upload(particles)
        self._time = float(time)
        self._step_count = int(step)
        self._frame_index = int(frame)
        self._mass_eps = float(mass_eps)
        lib().ckg_set_mass_epsilon(self._ctx, self._mass_eps)
        self._refresh_velocity_stats(particles)

    # -- accessors ------------------------------------------------------
    def config(self) -> SceneConfig:
        return self.cfg

    def grid(self) -> GridFacade:
        return GridFacade(self)

    def time(self) -> float:
        return self._time

    def step_count(self) -> int:
        return self._step_count

    def frame_index(self) -> int:
        return self._frame_index

    def mass_epsilon(self) -> float:
        return self._mass_eps

    def timers(self) -> PhaseTimers:
        return self._timers

    def reset_timers(self):
        self._timers = PhaseTimers()

    def counters(self) -> TransferCounters:
        return self._counters

    def reset_counters(self):
        self._counters = TransferCounters()

    def fused(self) -> bool:
        """True when substeps run the fused G2P2G kernel (ckg_fused)."""
        return bool(lib().ckg_fused(self._ctx))

    def last_sort_kind(self) -> int:
        """0 full radix sort, 1 identity (no key changed), 2 incremental merge."""
        return getattr(self, "_last_sort_kind", 0)

    def particle_count(self) -> int:
        return self._n

    # -- stepping -------------------------------------------------------
    def _absorb(self, out: abi.StepOut, nsteps: int = 1):
        t = self._timers
        t.sort_s += out.phase_ms[0] * 1e-3
        t.activate_s += out.phase_ms[1] * 1e-3
        t.clear_s += out.phase_ms[2] * 1e-3
        t.p2g_s += out.phase_ms[3] * 1e-3
        t.grid_s += out.phase_ms[4] * 1e-3
        t.g2p_s += out.phase_ms[5] * 1e-3
        t.substeps += nsteps
        c = self._counters
        c.p2g_node_visits += out.p2g_node_visits * nsteps
        c.g2p_node_visits += out.g2p_node_visits * nsteps
        c.p2g_transfers += out.p2g_transfers * nsteps
        c.g2p_transfers += out.g2p_transfers * nsteps
        self._vmax = float(out.vmax)
        self._min_j = [float(out.min_j[m]) for m in range(len(self.cfg.materials))]
        self.last_active_blocks = int(out.active_blocks)
        self._last_sort_kind = int(out.sort_kind)

    def step(self, dt: float) -> abi.StepOut:
        """Simulation::step (simulation.hpp:150-188) on the device."""
        out = abi.StepOut()
        rc = lib().ckg_step(self._ctx, float(dt), C.byref(out))
        _raise_for(self._ctx, rc, out)
        self._absorb(out)
        self._time = float(self._T(self._time) + self._T(dt))
        self._step_count += 1
        return out

    def step_many(self, dt: float, count: int) -> abi.StepOut:
        """`count` substeps of fixed dt, enqueued back to back (one host sync)."""
        out = abi.StepOut()
        done = 0
        while done < count:
            k = min(255, count - done)
            rc = lib().ckg_step_many(self._ctx, float(dt), k, C.byref(out))
            # the completed substeps count also when a later one failed (the
            # reference's state advances substep by substep)
            ok = int(out.substeps_done)
            if ok:
                self._absorb(out, ok)
            for _ in range(ok):
                self._time = float(self._T(self._time) + self._T(dt))
            self._step_count += ok
            _raise_for(self._ctx, rc, out)
            done += k
        return out

    def step_phases(self, dt: float, stop_after: int) -> abi.StepOut:
        out = abi.StepOut()
        rc = lib().ckg_step_phases(self._ctx, float(dt), int(stop_after), C.byref(out))
        _raise_for(self._ctx, rc, out)
        return out

    def cfl_dt(self, remaining: float) -> float:
        """cfl_dt (simulation.hpp:134-145) with sound speeds (:73-81), in T."""
        T = self._T
        cmax = T(0)
        for mi, m in enumerate(self.cfg.materials):
            if m.is_fluid:
                c = T(np.sqrt(T(m.bulk) * T(m.gamma) * T(np.power(T(self._min_j[mi]), T(1) - T(m.gamma)))
                              / T(m.density)))
            else:
                c = T(np.sqrt((T(m.lam) + T(2) * T(m.mu)) / T(m.density)))
            cmax = c if cmax < c else cmax
        vmax = T(self._vmax)
        denom = cmax if vmax < cmax else vmax
        dt = T(self.cfg.cfl) * self.cfg.dx(self.precision) / denom if denom > 0 else T(remaining)
        if T(self.cfg.max_dt) > 0:
            dt = min(dt, T(self.cfg.max_dt))
        return float(min(dt, T(remaining)))

    def advance_frame(self, cb: Optional[Callable[["Simulation", float], None]] = None,
                      device: bool = True) -> int:
        """advance_frame (simulation.hpp:193-211); returns the substeps taken.

        Without a per-substep callback the whole frame runs on the device
        (ckg_advance_frame: CUDA graph, device cfl_dt, no host round trip per
        substep); with one (or device=False) this host loop over step() runs."""
        if cb is None and device:
            return self._advance_frame_device()
        T = self._T
        frame_dt = T(self.cfg.frame_dt)
        frame_end = frame_dt * T(self._frame_index + 1)
        steps = 0
        while True:
            rem = frame_end - T(self._time)
            if rem <= frame_dt * T(1e-9):
                self._time = float(frame_end)
                break
            dt = self.cfl_dt(float(rem))
            self.step(dt)
            if cb is not None:
                cb(self, dt)
            steps += 1
            if steps > self.cfg.max_substeps_per_frame:
                raise NumericalError(f"substep limit exceeded within one frame at t = {self._time:.6f}")
        self._frame_index += 1
        return steps

    def _advance_frame_device(self) -> int:
        fin = abi.FrameIn()
        fin.time = self._time
        fin.frame_dt = float(self._T(self.cfg.frame_dt))
        fin.frame_index = self._frame_index
        fin.cfl = float(self._T(self.cfg.cfl))
        fin.max_dt = float(self._T(self.cfg.max_dt))
        fin.max_substeps = int(self.cfg.max_substeps_per_frame)
        fin.vmax = self._vmax
        for m in range(abi.MAX_MATERIALS):
            fin.min_j[m] = self._min_j[m] if m < len(self._min_j) else 1.0
        out = abi.FrameOut()
        rc = lib().ckg_advance_frame(self._ctx, C.byref(fin), C.byref(out))
        # bookkeeping of the completed substeps, also when a later one failed
        self._time = float(out.time)
        self._step_count += int(out.substeps)
        self._timers.substeps += int(out.substeps)
        # node visits per particle (transfer.hpp:32-45): compact 2 x 8 (MLS
        # scatters twice), quadratic baseline 27
        quad = self.cfg.kernel == "quadratic"
        per = 27 if quad else 32 if self.cfg.scheme == "mls" else 16
        c = self._counters
        c.p2g_node_visits += per * self._n * int(out.substeps)
        c.g2p_node_visits += (27 if quad else 16) * self._n * int(out.substeps)
        c.p2g_transfers += self._n * int(out.substeps)
        c.g2p_transfers += self._n * int(out.substeps)
        self._vmax = float(out.vmax)
        self._min_j = [float(out.min_j[m]) for m in range(len(self.cfg.materials))]
        if rc != abi.OK:
            so = abi.StepOut()
            so.error_code = out.error_code
            so.error_particle = out.error_particle
            _raise_for(self._ctx, rc, so)
        self._frame_index += 1
        self.last_frame = out
        return int(out.substeps)

    def diagnostics(self) -> DiagnosticsRow:
        """compute_diagnostics (simulation.hpp:55-69) as a device reduction."""
        d = abi.Diagnostics()
        _raise_for(self._ctx, lib().ckg_diagnostics_compute(self._ctx, C.byref(d)))
        return DiagnosticsRow(self._step_count, self._time, np.array(d.momentum[:]), np.array(d.angular[:]),
                              np.array(d.momentum_massfree[:]), float(d.kinetic_energy), float(d.vmax))

    # -- checkpoint / snapshot (io.hpp:344-477) ---------------------------
    def _records(self, kind: int) -> np.ndarray:
        """Device-packed file body (ckg_pack_records), one record per particle."""
        nb = int(lib().ckg_record_bytes(self._ctx, kind))
        buf = np.empty(self._n * nb, dtype=np.uint8)
        _raise_for(self._ctx, lib().ckg_pack_records(self._ctx, kind, abi.ptr(buf), buf.nbytes, 0))
        return buf

    def write_checkpoint(self, path: str):
        """write_checkpoint (io.hpp:392-430), CKCHKPT1, byte-identical layout."""
        import struct
        T = self._T
        head = b"CKCHKPT1" + struct.pack("<IQi", np.dtype(T).itemsize, self._step_count, self._frame_index)
        head += np.array([self._time, self._mass_eps], dtype=T).tobytes() + struct.pack("<Q", self._n)
        with open(path, "wb") as f:
            f.write(head)
            f.write(self._records(abi.RECORDS_CHECKPOINT).tobytes())

    def read_checkpoint(self, path: str):
        """read_checkpoint (io.hpp:432-477) into this simulation (restore)."""
        import struct
        T = self._T
        ts = np.dtype(T).itemsize
        data = open(path, "rb").read()
        if data[:8] != b"CKCHKPT1":
            raise IoError(f"not a checkpoint file: {path}")
        (scalar,) = struct.unpack_from("<I", data, 8)
        if scalar != ts:
            raise IoError(f"checkpoint scalar width mismatch in {path}")
        step, frame = struct.unpack_from("<Qi", data, 12)
        time, eps = np.frombuffer(data, dtype=T, count=2, offset=24)
        (count,) = struct.unpack_from("<Q", data, 24 + 2 * ts)
        rec = np.dtype([("f", T, 27), ("mat", "<u4")])
        off = 32 + 2 * ts
        if len(data) < off + count * rec.itemsize:
            raise IoError(f"truncated checkpoint particle data: {path}")
        r = np.frombuffer(data, dtype=rec, count=count, offset=off)
        p = np.zeros(count, dtype=abi.particle_dtype(self.precision))
        p["x"], p["v"] = r["f"][:, 0:3], r["f"][:, 3:6]
        p["F"], p["B"] = r["f"][:, 6:15].reshape(-1, 3, 3), r["f"][:, 15:24].reshape(-1, 3, 3)
        p["J"], p["mass"], p["volume0"] = r["f"][:, 24], r["f"][:, 25], r["f"][:, 26]
        p["material"] = r["mat"]
        self.restore(p, float(time), int(step), int(frame), float(eps))

    def write_snapshot(self, path: str, frame: int, binary: bool = True):
        """write_snapshot_binary / _text (io.hpp:344-390): x, v, J (fluids) or
        det F, material; same bytes as the reference's writers."""
        import struct
        body = self._records(abi.RECORDS_SNAPSHOT)
        dx = float(self.cfg.dx(self.precision))
        t = float(self._T(self._time))
        if binary:
            with open(path, "wb") as f:
                f.write(b"CKSNAP1\0" + struct.pack("<qdqd", frame, t, self._n, dx))
                f.write(body.tobytes())
            return
        r = np.frombuffer(body, dtype=np.dtype([("c", "<f8", 7), ("mat", "<u4")]))
        lines = ["# ckmpm-snapshot-v1\n", f"frame {frame}\n", "time %.17g\n" % t, f"count {self._n}\n",
                 "dx %.17g\n" % dx, "# x y z vx vy vz J_or_detF material_id\n"]
        for c, m in zip(r["c"].tolist(), r["mat"].tolist()):
            lines.append("".join("%.17g " % v for v in c) + f"{m}\n")
        with open(path, "w") as f:
            f.write("".join(lines))

    # -- binning parity hooks -------------------------------------------
    def debug_sort(self):
        keys = np.zeros(self._n, dtype=np.uint32)
        order = np.zeros(self._n, dtype=np.uint32)
        _raise_for(self._ctx, lib().ckg_debug_sort(self._ctx, abi.ptr(keys), abi.ptr(order), self._n))
        return keys, order

    def debug_bases(self):
        b = np.zeros((self._n, 2, 3), dtype=np.int32)
        _raise_for(self._ctx, lib().ckg_debug_bases(self._ctx, abi.ptr(b), self._n))
        return b
