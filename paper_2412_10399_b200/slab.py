"""x-slab decomposition of the CK-MPM substep over several GPUs.

One process (rank) per GPU owns the block planes bx in [bx_lo, bx_hi) and
the particles whose sort key lies there.  The device work of a substep runs in
the library (libckmpm_b200.so, csrc/ckg_slab.cuh); between its stages this
module moves the exchange buffers:

  1. footprint flags of the planes shared with the neighbours (planes
     bx_lo-2..bx_lo from the left, bx_hi-1..bx_hi from the right), OR-merged:
     the block set, and so the block order, of every plane two neighbours
     share is identical on both, so a halo plane is one contiguous pool slice
     on either side (the rest of each rank's directory is local);
  2. after P2G: ghost planes (bx_lo-1, bx_hi) sent to their owners and added
     (halo reduce-add of mass + momentum, both grids);
  3. after the grid update: boundary planes sent back into the neighbours'
     ghost planes (halo broadcast of velocities);
  4. after G2P: migrant counts, then migrant records; each rank rebuilds
     [left migrants][survivors][right migrants], which the next substep's
     stable sort turns into the global stable order restricted to the slab
     (bit-identical binning and order to a single-domain run);
  5. vmax / min J all-reduced for the CFL step.

The substep is a generator (`SlabRank.stages`) that yields exchange requests,
so the same code runs over torch.distributed (NCCL on GPUs, gloo on CPU) or
in-process over several contexts on one GPU (`run_loopback`, used by the
tests: no kernel ever waits on another rank's kernel).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from .scene import SceneConfig, mass_epsilon, seed_particles, to_abi_config


# ------------------------------------------------------------- partitioning

def block_x_of(particles: np.ndarray, cfg: SceneConfig, precision: int = 8) -> np.ndarray:
    """Sort-key block x (simulation.hpp:256-261), exact in T."""
    T = np.float64 if precision == 8 else np.float32
    dx = cfg.dx(precision)
    inv_dx = T(1) / dx
    D = cfg.resolution // 4 + 2
    x = particles["x"][:, 0].astype(T)
    b = np.floor(x * inv_dx + T(0.25)).astype(np.int64) >> 2
    return np.clip(b, 0, D - 1)


def partition_planes(plane_counts: np.ndarray, world: int) -> List[int]:
    """Slab boundaries X_0=0 < X_1 < ... < X_world=D over block planes,
    balancing particle counts (prefix-sum split); every rank gets >= 1 plane."""
    D = len(plane_counts)
    if world > D:
        raise ValueError("more ranks than block planes")
    cum = np.concatenate([[0], np.cumsum(plane_counts)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        x = int(np.searchsorted(cum, target, side="left"))
        x = max(x, bounds[-1] + 1)
        x = min(x, D - (world - r))
        bounds.append(x)
    bounds.append(D)
    return bounds


def rebalanced_bounds(bounds: Sequence[int], plane_counts: np.ndarray, max_shift: int = 1) -> List[int]:
    """Slab bounds for the current particle distribution: the balanced
    partition (partition_planes), each interior boundary moved at most
    `max_shift` planes towards it (a rank's new slab then only overlaps its
    neighbours' old ones, so planes change hands through the ordinary
    neighbour migration) and every rank keeps at least one plane."""
    world = len(bounds) - 1
    target = partition_planes(plane_counts, world)
    out = [int(bounds[0])]
    for r in range(1, world):
        b = int(bounds[r])
        b = min(max(int(target[r]), b - max_shift), b + max_shift)
        b = max(b, out[-1] + 1)
        b = min(b, int(bounds[r + 1]) - 1 if r + 1 < world else int(bounds[world]) - 1)
        out.append(b)
    out.append(int(bounds[world]))
    return out


def split_particles(particles: np.ndarray, cfg: SceneConfig, world: int, precision: int = 8):
    """Global stable order by key (the reference's sort_particles), then the
    contiguous slab ranges of it.  Returns (bounds, [per-rank arrays])."""
    D = cfg.resolution // 4 + 2
    T = np.float64 if precision == 8 else np.float32
    dx = cfg.dx(precision)
    inv_dx = T(1) / dx
    c = np.clip(np.floor(particles["x"].astype(T) * inv_dx + T(0.25)).astype(np.int64) >> 2, 0, D - 1)
    key = (c[:, 0] * D + c[:, 1]) * D + c[:, 2]
    order = np.argsort(key, kind="stable")
    ps = particles[order]
    bx = c[order, 0]
    counts = np.bincount(bx, minlength=D)
    bounds = partition_planes(counts, world)
    parts = [ps[(bx >= bounds[r]) & (bx < bounds[r + 1])] for r in range(world)]
    return bounds, parts


# --------------------------------------------------------------- requests

@dataclass
class AllReduceMax:
    buf: object           # torch.Tensor (int32, device)


@dataclass
class AllReduceSum:
    buf: object           # torch.Tensor (int64, device): summed in place


@dataclass
class Neighbor:
    send_left: Optional[object]
    send_right: Optional[object]
    recv_left: Optional[object]
    recv_right: Optional[object]
    # True: the transport may leave the transfer in flight (NCCL: on a side
    # stream after the sends' producers) until the next Join
    overlap: bool = False


@dataclass
class Join:
    """The transfers left in flight by overlap Neighbor requests complete
    before the library's next kernels (NCCL: the library stream waits)."""


@dataclass
class Counts:
    """Exchange two integers with the neighbours: send (to_left, to_right),
    receive (from_left, from_right) into `out` (list of 2)."""
    to_left: int
    to_right: int
    out: list


@dataclass
class Scalars:
    """All-reduce [vmax, -minJ...] by max and error flags by max."""
    values: np.ndarray
    out: list


def _check(lib, ctx, rc, what):
    if rc != 0:
        buf = C.create_string_buffer(512)
        lib.ckg_last_error_message(ctx, buf, 512)
        raise RuntimeError(f"{what}: status {rc}: {buf.value.decode()}")


class SlabRank:
    """One rank of the x-slab decomposition (one ckg context, one GPU)."""

    def __init__(self, cfg: SceneConfig, rank: int, world: int, bounds: Sequence[int], particles: np.ndarray,
                 mass_eps: float, precision: int = 8, device: int = 0):
        import torch

        from ._lib import lib
        self.lib = lib()
        self.torch = torch
        self.cfg = cfg
        self.rank, self.world = rank, world
        self.bx_lo, self.bx_hi = int(bounds[rank]), int(bounds[rank + 1])
        self.bounds = [int(b) for b in bounds]
        self.substep = 0
        self.rebalance_every = 0
        self.precision = precision
        self.T = np.float64 if precision == 8 else np.float32
        self.tdtype = torch.float64 if precision == 8 else torch.float32
        self.device = torch.device("cuda", device)
        self._abi_cfg = to_abi_config(cfg, precision, mass_eps, device)
        ctx = C.c_void_p()
        rc = self.lib.ckg_create(C.byref(self._abi_cfg), C.byref(ctx))
        if rc != 0:
            raise RuntimeError(f"ckg_create failed ({rc})")
        self.ctx = ctx
        _check(self.lib, ctx, self.lib.ckg_slab_set(ctx, rank, world, self.bx_lo, self.bx_hi), "ckg_slab_set")
        p = np.ascontiguousarray(particles, dtype=abi.particle_dtype(precision))
        _check(self.lib, ctx, self.lib.ckg_upload(ctx, abi.ptr(p), len(p)), "ckg_upload")
        self.n = len(p)
        D = cfg.resolution // 4 + 2
        self.D = D
        self.core = torch.zeros(D * D * D, dtype=torch.int32, device=self.device)
        self.block_words = 512
        self.vel_words = 384  # 2 grids x 3 velocity components x 64 nodes
        self.rec_words = int(self.lib.ckg_slab_record_words())
        self.tile_words = int(self.lib.ckg_slab_tile_words())
        self.out = abi.StepOut()
        self.vmax = 0.0
        self.min_j = [1.0] * len(cfg.materials)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.ckg_destroy(self.ctx)
            self.ctx = None

    def _buf(self, blocks_or_recs: int, words: int):
        return self.torch.empty(max(1, blocks_or_recs) * words, dtype=self.tdtype, device=self.device)

    def stages(self, dt: float):
        """One substep; yields exchange requests (see module docstring).
        Every `rebalance_every` substeps (0: never) the slab bounds are first
        moved towards the balanced partition of the current particles
        (rebalanced_bounds); the planes that change hands travel with this
        substep's migrants."""
        lib, ctx = self.lib, self.ctx
        has_l, has_r = self.rank > 0, self.rank < self.world - 1
        self.substep += 1
        new_bounds = None
        if self.rebalance_every > 0 and self.substep % self.rebalance_every == 0 and self.world > 1:
            D = self.D
            counts = (C.c_uint64 * D)()
            _check(lib, ctx, lib.ckg_slab_plane_counts(ctx, counts), "ckg_slab_plane_counts")
            t = self.torch.tensor(np.frombuffer(counts, dtype=np.uint64).astype(np.int64), device=self.device)
            yield AllReduceSum(t)
            new_bounds = rebalanced_bounds(self.bounds, t.cpu().numpy().astype(np.float64))
            if new_bounds != list(self.bounds):
                _check(lib, ctx, lib.ckg_slab_rebound(ctx, new_bounds[self.rank], new_bounds[self.rank + 1]),
                       "ckg_slab_rebound")
            else:
                new_bounds = None
        _check(lib, ctx, lib.ckg_slab_bin(ctx, float(dt), C.c_void_p(self.core.data_ptr())), "ckg_slab_bin")
        # footprint flags of the planes shared with the neighbours (no global
        # all-reduce): the active set of a plane X (the one-block positive
        # halo, grid.hpp:137-139) needs the footprint flags of X - 1 and X,
        # which particles of key planes X - 2 .. X + 1 set.  This rank keeps
        # planes lo - 1 .. hi (own + ghosts) and so needs the left
        # neighbour's flags of lo - 2 .. lo and the right one's of
        # hi - 1 .. hi; each side's plane set is then identical on both
        # ranks, and so is its block order (halo messages match block for
        # block) while the rest of the directory stays local.
        D, PL = self.D, self.D * self.D

        def span(a, b):
            a, b = max(a, 0), min(b, D - 1)
            return (a, b) if a <= b else None

        def view(sp):
            return self.core[sp[0] * PL:(sp[1] + 1) * PL]

        sl_span = span(self.bx_lo - 1, self.bx_lo) if has_l else None  # -> left
        sr_span = span(self.bx_hi - 2, self.bx_hi) if has_r else None  # -> right
        rl_span = span(self.bx_lo - 2, self.bx_lo) if has_l else None  # <- left
        rr_span = span(self.bx_hi - 1, self.bx_hi) if has_r else None  # <- right
        send_l = view(sl_span).clone() if sl_span else None
        send_r = view(sr_span).clone() if sr_span else None
        recv_l = self.torch.empty_like(view(rl_span)) if rl_span else None
        recv_r = self.torch.empty_like(view(rr_span)) if rr_span else None
        yield Neighbor(send_l, send_r, recv_l, recv_r)
        if recv_l is not None:
            v = view(rl_span)
            v.copy_(self.torch.maximum(v, recv_l))
        if recv_r is not None:
            v = view(rr_span)
            v.copy_(self.torch.maximum(v, recv_r))
        # P2G: with neighbours, the two boundary planes first (the only ones
        # whose tiles reach the ghost planes), their halo then travels while
        # the interior planes scatter
        split = has_l or has_r
        planes = (C.c_uint64 * 4)()
        _check(lib, ctx, lib.ckg_slab_p2g_part(ctx, C.c_void_p(self.core.data_ptr()), planes, 1 if split else 0),
               "ckg_slab_p2g_part")
        pb = [int(v) for v in planes]  # blocks of planes ghostL, ownL, ownR, ghostR

        def interior_p2g():
            if split:
                _check(lib, ctx, lib.ckg_slab_p2g_part(ctx, None, (C.c_uint64 * 4)(), 2), "ckg_slab_p2g_part")

        W = self.block_words
        if self.cfg.deterministic:
            # the boundary planes' P2G tiles -> the neighbours' ghost planes;
            # each rank then sums its nodes over local and received tiles in
            # the single-domain order (ckg_slab_grid)
            TW = self.tile_words
            send_l = self._buf(pb[1], TW) if has_l else None
            send_r = self._buf(pb[2], TW) if has_r else None
            if send_l is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 3, 1, C.c_void_p(send_l.data_ptr())), "tile pack")
            if send_r is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 3, 2, C.c_void_p(send_r.data_ptr())), "tile pack")
            recv_l = self._buf(pb[0], TW) if has_l else None
            recv_r = self._buf(pb[3], TW) if has_r else None
            yield Neighbor(send_l, send_r, recv_l, recv_r, overlap=True)
            interior_p2g()
            yield Join()
            if recv_l is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 4, 0, C.c_void_p(recv_l.data_ptr())), "tile set")
            if recv_r is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 4, 3, C.c_void_p(recv_r.data_ptr())), "tile set")
        else:
            # halo reduce-add: ghost planes -> owners
            send_l = self._buf(pb[0], W) if has_l else None
            send_r = self._buf(pb[3], W) if has_r else None
            if send_l is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 0, 0, C.c_void_p(send_l.data_ptr())), "halo pack")
            if send_r is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 0, 3, C.c_void_p(send_r.data_ptr())), "halo pack")
            recv_l = self._buf(pb[1], W) if has_l else None
            recv_r = self._buf(pb[2], W) if has_r else None
            yield Neighbor(send_l, send_r, recv_l, recv_r, overlap=True)
            interior_p2g()  # (its flushes also add into the own boundary planes:
            yield Join()    # the received halo is added after it, on the same stream)
            if recv_l is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 1, 1, C.c_void_p(recv_l.data_ptr())), "halo add")
            if recv_r is not None:
                _check(lib, ctx, lib.ckg_slab_halo(ctx, 1, 2, C.c_void_p(recv_r.data_ptr())), "halo add")
        _check(lib, ctx, lib.ckg_slab_grid(ctx), "ckg_slab_grid")
        # halo broadcast of velocities (only: G2P reads no ghost masses): own
        # boundary planes -> neighbours' ghosts
        VW = self.vel_words
        send_l = self._buf(pb[1], VW) if has_l else None
        send_r = self._buf(pb[2], VW) if has_r else None
        if send_l is not None:
            _check(lib, ctx, lib.ckg_slab_halo(ctx, 5, 1, C.c_void_p(send_l.data_ptr())), "vel pack")
        if send_r is not None:
            _check(lib, ctx, lib.ckg_slab_halo(ctx, 5, 2, C.c_void_p(send_r.data_ptr())), "vel pack")
        recv_l = self._buf(pb[0], VW) if has_l else None
        recv_r = self._buf(pb[3], VW) if has_r else None
        yield Neighbor(send_l, send_r, recv_l, recv_r)
        if recv_l is not None:
            _check(lib, ctx, lib.ckg_slab_halo(ctx, 6, 0, C.c_void_p(recv_l.data_ptr())), "vel set")
        if recv_r is not None:
            _check(lib, ctx, lib.ckg_slab_halo(ctx, 6, 3, C.c_void_p(recv_r.data_ptr())), "vel set")
        # G2P and migration
        counts = (C.c_uint64 * 2)()
        _check(lib, ctx, lib.ckg_slab_g2p(ctx, counts), "ckg_slab_g2p")
        out_l, out_r = int(counts[0]), int(counts[1])
        if (out_l and not has_l) or (out_r and not has_r):
            raise RuntimeError("particle left the global domain through a slab edge")
        got = [0, 0]
        yield Counts(out_l, out_r, got)
        nl_in, nr_in = got
        R = self.rec_words
        send_l, send_r = self._buf(out_l, R), self._buf(out_r, R)
        _check(lib, ctx, lib.ckg_slab_pack(ctx, nl_in, C.c_void_p(send_l.data_ptr()), C.c_void_p(send_r.data_ptr())),
               "ckg_slab_pack")
        recv_l, recv_r = self._buf(nl_in, R), self._buf(nr_in, R)
        yield Neighbor(send_l[: out_l * R] if has_l else None, send_r[: out_r * R] if has_r else None,
                       recv_l[: nl_in * R] if has_l else None, recv_r[: nr_in * R] if has_r else None)
        rc = lib.ckg_slab_finish(ctx, C.c_void_p(recv_l.data_ptr()), nl_in, C.c_void_p(recv_r.data_ptr()), nr_in,
                                 C.byref(self.out))
        if new_bounds is not None:  # committed by ckg_slab_finish
            self.bounds = list(new_bounds)
            self.bx_lo, self.bx_hi = new_bounds[self.rank], new_bounds[self.rank + 1]
        # errors travel through the all-reduce below so every rank stops together
        self.out.status = rc
        self.n = self.n - out_l - out_r + nl_in + nr_in
        vals = np.array([self.out.vmax] + [-float(self.out.min_j[m]) for m in range(len(self.cfg.materials))]
                        + [float(self.out.status)], dtype=np.float64)
        red = [None]
        yield Scalars(vals, red)
        r = red[0]
        self.vmax = float(r[0])
        self.min_j = [-float(v) for v in r[1:1 + len(self.cfg.materials)]]
        if r[-1] != 0:
            buf = C.create_string_buffer(512)
            lib.ckg_last_error_message(ctx, buf, 512)
            raise RuntimeError(f"slab substep failed on some rank (local: {buf.value.decode() or 'ok'})")

    def particles(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=abi.particle_dtype(self.precision))
        _check(self.lib, self.ctx, self.lib.ckg_download(self.ctx, abi.ptr(out), self.n), "ckg_download")
        return out

    def cfl_dt(self, remaining: float) -> float:
        """cfl_dt (simulation.hpp:134-145) from the all-reduced vmax / min J."""
        T = self.T
        cmax = T(0)
        for mi, m in enumerate(self.cfg.materials):
            if m.is_fluid:
                c = T(np.sqrt(T(m.bulk) * T(m.gamma) * T(np.power(T(self.min_j[mi]), T(1) - T(m.gamma)))
                              / T(m.density)))
            else:
                c = T(np.sqrt((T(m.lam) + T(2) * T(m.mu)) / T(m.density)))
            cmax = c if cmax < c else cmax
        vmax = T(self.vmax)
        denom = cmax if vmax < cmax else vmax
        dt = T(self.cfg.cfl) * self.cfg.dx(self.precision) / denom if denom > 0 else T(remaining)
        if T(self.cfg.max_dt) > 0:
            dt = min(dt, T(self.cfg.max_dt))
        return float(min(dt, T(remaining)))


# ------------------------------------------------------------- transports

def run_loopback(ranks: List[SlabRank], dt: float):
    """Drive all ranks' stages in lock step inside one process (one GPU):
    exchanges are device-to-device copies between the ranks' buffers."""
    gens = [r.stages(dt) for r in ranks]
    world = len(ranks)
    while True:
        reqs = []
        done = False
        for g in gens:
            try:
                reqs.append(next(g))
            except StopIteration:
                done = True
        if done:
            assert len(reqs) == 0, "ranks out of step"
            return
        kind = type(reqs[0])
        assert all(type(q) is kind for q in reqs), "ranks out of step"
        # the library kernels that produced the send buffers run on the
        # contexts' own streams, the copies below on torch's
        ranks[0].torch.cuda.synchronize()
        if kind is Join:
            continue
        if kind is AllReduceSum:
            acc = reqs[0].buf.clone()
            for q in reqs[1:]:
                acc = acc + q.buf
            for q in reqs:
                q.buf.copy_(acc)
        elif kind is AllReduceMax:
            acc = reqs[0].buf.clone()
            for q in reqs[1:]:
                acc = ranks[0].torch.maximum(acc, q.buf)
            for q in reqs:
                q.buf.copy_(acc)
        elif kind is Neighbor:
            for r, q in enumerate(reqs):
                if r > 0 and q.recv_left is not None:
                    q.recv_left.copy_(reqs[r - 1].send_right)
                if r < world - 1 and q.recv_right is not None:
                    q.recv_right.copy_(reqs[r + 1].send_left)
        elif kind is Counts:
            for r, q in enumerate(reqs):
                q.out[0] = reqs[r - 1].to_right if r > 0 else 0
                q.out[1] = reqs[r + 1].to_left if r < world - 1 else 0
        elif kind is Scalars:
            m = np.max(np.stack([q.values for q in reqs]), axis=0)
            for q in reqs:
                q.out[0] = m
        # torch copies run on torch's stream; the library on its own
        ranks[0].torch.cuda.synchronize()


class DistTransport:
    """torch.distributed transport (NCCL for device buffers; works with gloo
    for CPU tensors too).  Neighbours are rank-1 / rank+1 (no wrap)."""

    def __init__(self, dist, rank: int, world: int, device):
        self.dist, self.rank, self.world, self.device = dist, rank, world, device
        # gloo cannot move CUDA tensors point-to-point: stage through host
        # memory (used to run several ranks on one GPU in tests)
        self.host_staged = dist.get_backend() == "gloo" and getattr(device, "type", "cpu") == "cuda"
        self.comm_device = "cpu" if self.host_staged else device
        self.pending = []  # works of overlap Neighbor requests (until Join)
        self._side = None

    def _side_stream(self):
        import torch
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _out(self, t):
        return t.cpu() if (self.host_staged and t is not None) else t

    def handle(self, req):
        import torch
        d = self.dist
        if isinstance(req, AllReduceSum):
            buf = self._out(req.buf)
            d.all_reduce(buf, op=d.ReduceOp.SUM)
            if buf is not req.buf:
                req.buf.copy_(buf)
        elif isinstance(req, AllReduceMax):
            buf = self._out(req.buf)
            d.all_reduce(buf, op=d.ReduceOp.MAX)
            if buf is not req.buf:
                req.buf.copy_(buf)
        elif isinstance(req, Neighbor):
            sl, sr = self._out(req.send_left), self._out(req.send_right)
            rl, rr = self._out(req.recv_left), self._out(req.recv_right)
            ops = []
            if self.rank > 0:
                if sl is not None:
                    ops.append(d.P2POp(d.isend, sl.contiguous(), self.rank - 1))
                if rl is not None:
                    ops.append(d.P2POp(d.irecv, rl, self.rank - 1))
            if self.rank < self.world - 1:
                if sr is not None:
                    ops.append(d.P2POp(d.isend, sr.contiguous(), self.rank + 1))
                if rr is not None:
                    ops.append(d.P2POp(d.irecv, rr, self.rank + 1))
            ops = [o for o in ops if o.tensor.numel() > 0]
            if req.overlap and ops and not self.host_staged and torch.cuda.is_available():
                # in flight on a side stream (ordered after the packing
                # kernels) while the library enqueues its next kernels; Join
                # makes the library stream wait for it
                cur = torch.cuda.current_stream(self.device)
                side = self._side_stream()
                side.wait_stream(cur)
                with torch.cuda.stream(side):
                    self.pending.extend(d.batch_isend_irecv(ops))
                return
            if ops:
                for w in d.batch_isend_irecv(ops):
                    w.wait()
            if rl is not None and rl is not req.recv_left:
                req.recv_left.copy_(rl)
            if rr is not None and rr is not req.recv_right:
                req.recv_right.copy_(rr)
        elif isinstance(req, Join):
            for w in self.pending:
                w.wait()  # NCCL: the current (library) stream waits, not the host
            self.pending = []
        elif isinstance(req, Counts):
            t = torch.tensor([req.to_left, req.to_right], dtype=torch.int64, device=self.comm_device)
            allc = [torch.zeros(2, dtype=torch.int64, device=self.comm_device) for _ in range(self.world)]
            d.all_gather(allc, t)
            req.out[0] = int(allc[self.rank - 1][1]) if self.rank > 0 else 0
            req.out[1] = int(allc[self.rank + 1][0]) if self.rank < self.world - 1 else 0
        elif isinstance(req, Scalars):
            t = torch.tensor(req.values, dtype=torch.float64, device=self.comm_device)
            d.all_reduce(t, op=d.ReduceOp.MAX)
            req.out[0] = t.cpu().numpy()

    def step(self, rank_obj: SlabRank, dt: float):
        import torch
        import os
        host_sync = os.environ.get("CKMPM_SLAB_HOST_SYNC", "0") == "1"  # round-1 behaviour, a fallback switch
        if self.host_staged or host_sync or not torch.cuda.is_available():
            for req in rank_obj.stages(dt):
                # the library runs on its own (non-blocking) stream: its send
                # buffers are complete before the host reads them, and the
                # received data is visible before control returns to it
                if torch.cuda.is_available():
                    torch.cuda.synchronize()
                self.handle(req)
                if torch.cuda.is_available():
                    torch.cuda.synchronize()
            return
        # NCCL: every exchange is enqueued on the library's own stream (the
        # process group orders its communication stream after it and the
        # stream after the transfer), so packing kernel -> send/recv -> the
        # kernels consuming the halo are ordered on the device; the host only
        # waits where the library itself needs a count
        ext = torch.cuda.ExternalStream(rank_obj.lib.ckg_stream(rank_obj.ctx), device=self.device)
        with torch.cuda.stream(ext):
            for req in rank_obj.stages(dt):
                self.handle(req)


def build_ranks(cfg: SceneConfig, world: int, precision: int = 8, particles: Optional[np.ndarray] = None,
                devices: Optional[Sequence[int]] = None, only_rank: Optional[int] = None):
    """Seed (or take) the global particle set, split it into slabs and build
    the rank objects (all of them for loopback, one for a real rank)."""
    p = seed_particles(cfg, precision) if particles is None else particles
    me = mass_epsilon(p, precision)  # global median, as the single-domain run
    bounds, parts = split_particles(p, cfg, world, precision)
    # refresh_velocity_stats (simulation.hpp:234-243) over the global set
    T = np.float64 if precision == 8 else np.float32
    v = p["v"].astype(T)
    vmax = float(np.max(np.sqrt((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2]))) if len(p) else 0.0
    min_j = [1.0] * len(cfg.materials)
    for mi, m in enumerate(cfg.materials):
        sel = p["J"][p["material"] == mi]
        if m.is_fluid and len(sel):
            min_j[mi] = min(1.0, float(np.min(sel)))
    ranks = []
    for r in range(world):
        if only_rank is not None and r != only_rank:
            continue
        dev = devices[r] if devices else 0
        rk = SlabRank(cfg, r, world, bounds, parts[r], me, precision, dev)
        rk.vmax, rk.min_j = vmax, list(min_j)
        ranks.append(rk)
    return bounds, ranks


def _lattice_i_extent(cfg: SceneConfig, precision: int):
    """Outer (x) cell range of every body's lattice sampler (scene.hpp:85-88)."""
    import math

    from .scene import _aabb
    T = np.float64 if precision == 8 else np.float32
    dx = cfg.dx(precision)
    lo, hi = None, None
    for b in cfg.bodies:
        blo, bhi = _aabb(b.shape, T)
        i0 = int(math.floor(T(blo[0]) / dx)) - 1
        i1 = int(math.ceil(T(bhi[0]) / dx)) + 1
        lo = i0 if lo is None else min(lo, i0)
        hi = i1 if hi is None else max(hi, i1)
    return lo, hi


def scene_marginals(cfg: SceneConfig, precision: int = 8, chunk_cells: int = 16):
    """Particles per sort-key block plane, the (mass, count) multiset and the
    largest initial speed of the whole scene, by seeding it in chunks of x
    cells (every rank can compute them without holding the particle set)."""
    T = np.float64 if precision == 8 else np.float32
    D = cfg.resolution // 4 + 2
    counts = np.zeros(D, dtype=np.int64)
    masses = {}
    vmax2 = T(0)
    lattice = all(b.ppc in (8, 27) for b in cfg.bodies)
    lo, hi = _lattice_i_extent(cfg, precision)
    ranges = [(a, min(a + chunk_cells - 1, hi)) for a in range(lo, hi + 1, chunk_cells)] if lattice else [None]
    for r in ranges:
        p = seed_particles(cfg, precision, i_range=r, allow_empty=True)
        if len(p) == 0:
            continue
        counts += np.bincount(block_x_of(p, cfg, precision), minlength=D)
        m, c = np.unique(p["mass"], return_counts=True)
        for mv, cv in zip(m.tolist(), c.tolist()):
            masses[mv] = masses.get(mv, 0) + cv
        v = p["v"].astype(T)
        s2 = (v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2]
        vmax2 = max(vmax2, T(np.max(s2)))
    return counts, masses, float(np.sqrt(vmax2))


def _median_mass_eps(masses: dict, precision: int) -> float:
    """compute_mass_epsilon (simulation.hpp:227-232, nth_element at n/2) over a
    (mass, count) multiset."""
    T = np.float64 if precision == 8 else np.float32
    n = sum(masses.values())
    k = n // 2
    run = 0
    for m in sorted(masses):
        run += masses[m]
        if run > k:
            return float(T(1e-12) * T(m))
    raise ValueError("no particles")


def build_rank_local(cfg: SceneConfig, world: int, rank: int, precision: int = 8, device: int = 0):
    """Rank-local seeding for any scene of lattice bodies (ppc 8 / 27;
    jittered ppc 16 bodies are seeded whole and filtered): slab bounds from
    the x-marginal of the scene (scene_marginals), then each rank seeds only
    the lattice x-cells whose particles can have their sort-key plane in its
    slab and keeps those that do.  The seeding order restricted to a slab is
    the global emission order restricted to it (bodies in order, each i-major),
    so the first substep's stable sort gives exactly the slab's part of the
    global stable order; mass_eps and the initial vmax are the global ones."""
    bounds, part, me, vmax = rank_local_particles(cfg, world, rank, precision)
    rk = SlabRank(cfg, rank, world, bounds, part, me, precision, device)
    rk.vmax = vmax
    # (seeded J = 1: min J of every material stays 1)
    return bounds, rk


def rank_local_particles(cfg: SceneConfig, world: int, rank: int, precision: int = 8):
    """(bounds, this rank's particles in seeding order, global mass_eps,
    global initial vmax) -- see build_rank_local."""
    counts, masses, vmax = scene_marginals(cfg, precision)
    bounds = partition_planes(counts.astype(np.float64), world)
    lo, hi = bounds[rank], bounds[rank + 1]
    # key plane X <=> x/dx + 1/4 in [4X, 4X + 4): cells 4 lo - 1 .. 4 hi
    part = seed_particles(cfg, precision, i_range=(4 * lo - 1, 4 * hi), allow_empty=True)
    if len(part):
        kbx = block_x_of(part, cfg, precision)
        part = part[(kbx >= lo) & (kbx < hi)]
    return bounds, part, _median_mass_eps(masses, precision), vmax


# the bench's single-box scenes (kept name)
build_rank_for_box = build_rank_local
