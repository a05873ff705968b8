#!/usr/bin/env python3
"""CK-MPM per-substep transfer benchmark (BASELINE.json metric:
particle-substeps/s and P2G+G2P HBM roofline) on B200.

Default workload (N=1): SURVEY Appendix C `C5_block_108` — fixed-corotated
block of 108^3 cells at 8 ppc (10,077,696 particles), res 512, APIC, sticky
floor, gravity -9.8, FP64 (the reference's Simulation<double>).  One "step"
is one full substep (sort, activate, clear, P2G, grid update, G2P) at the
fixed dt = cfl_dt(t=0) (the replayed schedule of the reference's
`ckmpm bench`, proj/tools/ckmpm_main.cpp:146-159).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 runs under torchrun, one process per GPU (see DESIGN.md §6 for the
multi-GPU status).  The particle state (2.26 GB) exceeds L2 (126 MB), so no
explicit flush is needed between substeps.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2412_10399_b200 import abi  # noqa: E402
from paper_2412_10399_b200.scene import block_scene, seed_particles  # noqa: E402

METRIC = "particle-substeps/s"
UNIT = "particle-substeps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=108, help="C5 block edge in cells (108 -> 10.08M p)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak (~10M particles per GPU) or strong (the fixed --strong-cells block)")
    ap.add_argument("--strong-cells", type=int, default=232, help="strong-scaling block edge (232 -> 99.9M p)")
    ap.add_argument("--model", default="fixed_corotated", choices=["fixed_corotated", "drucker_prager"],
                    help="block material (drucker_prager: the sand scene of the north star's scaling target)")
    ap.add_argument("--force-slab", action="store_true",
                    help="testing: run the x-slab path even at N=1 (one slab, NCCL process group of one)")
    ap.add_argument("--rebalance-every", type=int, default=0,
                    help="N>1: move the slab bounds towards balance every K substeps (0: never)")
    ap.add_argument("--res", type=int, default=512)
    ap.add_argument("--scheme", default="apic")
    ap.add_argument("--kernel", default="compact", choices=["compact", "quadratic"],
                    help="quadratic: the 27-node B-spline baseline (paper's comparison)")
    ap.add_argument("--precision", type=int, default=8, choices=[8, 4])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chains", type=int, default=3,
                    help="secondary e2e figure: independent host-resident simulations stepped concurrently "
                         "(one host thread each); the headline e2e is one simulation")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fused", action="store_true",
                    help="fused G2P2G kernel instead of the separate P2G / G2P kernels (CKG_FLAG_FUSED)")
    ap.add_argument("--no-single", action="store_true",
                    help="skip the secondary FP32 (Simulation<float>) device-rate figure")
    ap.add_argument("--cpu-cells", type=int, default=None,
                    help="CPU baseline block edge (default: the bench's own --cells, i.e. the same config)")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--cpu-det-steps", type=int, default=1,
                    help="CPU baseline: substeps also timed in the reference's deterministic (serial scatter) mode")
    ap.add_argument("--ref-warmup", type=int, default=1, help="reference arm: untimed substeps before timing")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: bound on the timed substeps' wall time (N>1 workloads)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        load = [s for s in sm if s is not None]
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def algorithmic_bytes(n, nblocks, scheme, precision):
    """SURVEY §8(d) compulsory bytes per launch for the reference semantics
    (stress recomputed in P2G, sort applied through the G2P writes):
    P2G reads x, v, F, B, m, V0, mat (FP64 APIC 212 B/particle; PIC -72 B)
    and writes every active node once (2 grids x 64 nodes x {m, p} = 32 B/node);
    G2P reads x, F, mat (100 B) and writes x, v, F, B (192 B; PIC -72 B),
    plus the nodal velocities (24 B/node).  The implementation's own choices
    (stress cache, full-state rewrite) are not counted: profiles/traffic.json
    holds what the kernels actually move."""
    s = precision
    b = 9 * s if scheme != "pic" else 0
    nodes = nblocks * 2 * 64
    p2g = n * (3 * s + 3 * s + 9 * s + b + s + s + 4) + nodes * 4 * s
    g2p = n * (3 * s + 9 * s + 4) + n * (3 * s + 3 * s + 9 * s + b) + nodes * 3 * s
    return p2g, g2p


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def single_precision_rate(args, cfg, local):
    """The same scene and substep in the reference's single-precision mode
    (`ckmpm run --precision single`, tools/ckmpm_main.cpp:122): device time of
    K substeps after W warm-up ones, CUDA events on the library stream."""
    from paper_2412_10399_b200._lib import lib
    from paper_2412_10399_b200.api import Simulation

    L = lib()
    host = seed_particles(cfg, 4)
    sim = Simulation(cfg, precision=4, device=local, particles=host, fused=True if args.fused else None)
    fused = sim.fused()
    ctx = sim._ctx
    dt = sim.cfl_dt(1.0)
    o = abi.StepOut()
    for _ in range(args.warmup):
        assert L.ckg_step(ctx, dt, C.byref(o)) == 0
    acc = [0.0] * 6
    L.ckg_timer_mark(ctx, 0)
    for _ in range(args.steps):
        assert L.ckg_step(ctx, dt, C.byref(o)) == 0
        for k in range(6):
            acc[k] += o.phase_ms[k] / args.steps
    L.ckg_timer_mark(ctx, 1)
    el = C.c_double()
    L.ckg_timer_elapsed(ctx, 0, 1, C.byref(el))
    sim.close()
    n = len(host)
    return {"value": n * args.steps / (el.value * 1e-3), "unit": UNIT, "dtype": "f32", "fused": fused,
            "ms_per_step": el.value / args.steps, "phase_ms": dict(zip(abi.PHASE_NAMES, acc)),
            "parity": "keys/order bit-exact and state <= 1e-5 vs the reference's Simulation<float> "
                      "(tests/test_gpu_parity.py::test_float_mode_vs_reference_float)"}


def cpu_cells(args):
    return workload_cells(args, 1) if args.cpu_cells is None else args.cpu_cells


def cpu_baseline(args, threads):
    """Reference engine (oracle/_ref, compiled unmodified) on the host cores:
    Simulation<double>::step on the bench's own scene (same config; a bounded
    number of substeps), atomic (default) mode."""
    from oracle import bind
    cfg = bench_scene(args, cpu_cells(args))
    p = seed_particles(cfg, args.precision)
    ref = bind.Ref(cfg, p, precision=args.precision, threads=threads, deterministic=False)
    dt = ref.cfl_dt(1.0)
    rc, msg = ref.step(dt)  # warm-up (allocations, first touch)
    if rc:
        raise RuntimeError(msg)
    t0 = time.perf_counter()
    for _ in range(args.cpu_steps):
        rc, msg = ref.step(dt)
        if rc:
            raise RuntimeError(msg)
    el = time.perf_counter() - t0
    ref.close()
    det = None
    if args.cpu_det_steps > 0:
        # the reference's other mode (SimConfig::deterministic: serial scatter,
        # simulation.hpp:326-327), reported beside the default
        ref = bind.Ref(cfg, p, precision=args.precision, threads=threads, deterministic=True)
        t0 = time.perf_counter()
        for _ in range(args.cpu_det_steps):
            rc, msg = ref.step(dt)
            if rc:
                raise RuntimeError(msg)
        det = {"value": len(p) * args.cpu_det_steps / (time.perf_counter() - t0), "unit": UNIT,
               "steps": args.cpu_det_steps, "mode": "deterministic (serial scatter)"}
        ref.close()
    kind = "reference"
    return {"value": len(p) * args.cpu_steps / el, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"C5 block {cpu_cells(args)}^3 cells ({len(p)} p) res {args.res} {args.scheme} "
                      f"FP{8 * args.precision}, {args.cpu_steps} substeps after 1 warm-up, "
                      f"ckmpm::Simulation<T>::step (atomic P2G), wall clock",
            "deterministic": det}


def bench_scene(args, cells):
    """The C5 block of `cells`^3 cells; --model drucker_prager: the same block
    of sand (E 1e4, rho 1400, phi 30 deg as SURVEY App. C's C3/C4, separating
    floor, gravity -2)."""
    if args.model == "drucker_prager":
        return block_scene(cells, resolution=args.res, scheme=args.scheme, kernel=args.kernel,
                           model="drucker_prager", E=1e4, density=1400.0, gravity=(0, -2.0, 0),
                           boundary="separate")
    return block_scene(cells, resolution=args.res, scheme=args.scheme, kernel=args.kernel)


def workload_cells(args, ws):
    """Block edge of the workload at N GPUs: weak scaling (default) keeps the
    C5 block at N=1 and grows it so every GPU keeps ~10M particles; strong
    scaling runs the fixed --strong-cells block at every N."""
    if args.scaling == "strong":
        return args.strong_cells
    return args.cells if ws == 1 else int(round(args.cells * ws ** (1.0 / 3.0)))


def bench_config(args, cells, n, dt, nblocks=None):
    """The `config` object both arms print (same keys, same values)."""
    name = f"C5_block_{cells}" if args.model == "fixed_corotated" else f"sand_block_{cells}"
    return {"workload": name, "particles": n, "resolution": args.res, "kernel": args.kernel,
            "scheme": args.scheme, "material": args.model, "ppc": 8, "dt": dt,
            "active_blocks": nblocks, "l2": "state >> 126 MB L2 (no flush needed)"}


def run_reference(args):
    """Reference arm: the reference's own CPU engine (oracle/_ref: the
    unmodified ckmpm headers) on the same workload, all host threads, atomic
    (default) P2G.  Under torchrun only rank 0 runs it.  When the workload is
    too large for K substeps to finish within a few minutes (N > 1 weak
    scaling), the timed substeps are bounded (reported in `steps`)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import bind
    cells = workload_cells(args, ws)
    cfg = bench_scene(args, cells)
    p = seed_particles(cfg, args.precision)
    ref = bind.Ref(cfg, p, precision=args.precision, threads=threads, deterministic=False)
    dt = ref.cfl_dt(1.0)
    # the CPU engine needs no GPU-style warm-up (no clocks, caches or JIT to
    # settle); one untimed substep covers first-touch allocation
    t_w = time.perf_counter()
    for _ in range(max(1, min(args.warmup, args.ref_warmup))):
        rc, msg = ref.step(dt)
        assert rc == 0, msg
    t_one = (time.perf_counter() - t_w) / max(1, min(args.warmup, args.ref_warmup))
    steps = max(1, min(args.steps, int(args.ref_budget_s / max(t_one, 1e-9))))
    t0 = time.perf_counter()
    for _ in range(steps):
        rc, msg = ref.step(dt)
        assert rc == 0, msg
    el = time.perf_counter() - t0
    val = len(p) * steps / el
    tm = ref.timers()
    nblocks = ref.active_blocks()
    sample = (f"C5 block {cells}^3 cells ({len(p)} p) res {args.res} {args.scheme} FP{8 * args.precision}; "
              f"ckmpm::Simulation<T>::step, atomic P2G, {threads} threads, {steps} timed substeps")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": steps,
            "warmup": args.warmup, "ms_per_step": el / steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if args.precision == 8 else "f32",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(args, cells, len(p), dt, nblocks),
            "parallelism": f"cpu threads={threads}",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "phase_s": dict(zip(abi.PHASE_NAMES, tm))}
    print(json.dumps(line), flush=True)


def run_slab(args, ws, rank, local):
    """N>1: x-slab decomposition (paper_2412_10399_b200/slab.py), one rank
    per GPU over NCCL, every exchange ordered on the library's stream.
    Weak scaling (default): the C5 block grows with N so every GPU keeps ~10M
    particles (cells = 108 * N^(1/3)); strong (--scaling strong): the fixed
    --strong-cells block (232: 99.9M particles) split over the N GPUs.  Each
    rank seeds only its own slab (build_rank_local)."""
    import torch
    import torch.distributed as dist

    from paper_2412_10399_b200._lib import lib
    from paper_2412_10399_b200.slab import DistTransport, build_rank_local

    # CKMPM_BENCH_BACKEND=gloo: the same path with host-staged exchanges and
    # every rank on the GPUs present (tests on a single GPU; not a bench value)
    backend = os.environ.get("CKMPM_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    L = lib()
    dev = f"cuda:{local}"
    cells = workload_cells(args, ws)
    cfg = bench_scene(args, cells)
    bounds, rk = build_rank_local(cfg, ws, rank, args.precision, local)
    rk.rebalance_every = args.rebalance_every
    tr = DistTransport(dist, rank, ws, torch.device("cuda", local))
    n_local = torch.tensor([rk.n], dtype=torch.int64, device=dev)
    dist.all_reduce(n_local)
    n_total = int(n_local.item())
    dt = rk.cfl_dt(1.0)
    for _ in range(args.warmup):
        tr.step(rk, dt)
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    L.ckg_timer_mark(rk.ctx, 0)
    launches = 0
    phase = np.zeros(6)
    for _ in range(args.steps):
        tr.step(rk, dt)
        launches += int(rk.out.kernel_launches)
        phase += np.array(list(rk.out.phase_ms)) / args.steps
    L.ckg_timer_mark(rk.ctx, 1)
    el = C.c_double()
    L.ckg_timer_elapsed(rk.ctx, 0, 1, C.byref(el))
    clocks = sampler.stop()
    t = torch.tensor([el.value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    value = n_total * args.steps / (t_ms * 1e-3)
    # roofline of the slowest rank's transfer kernels: algorithmic bytes of
    # its own particles / blocks over its own P2G and G2P device times
    p2g_b, g2p_b = algorithmic_bytes(rk.n, int(rk.out.active_blocks), args.scheme, args.precision)
    peak, peak_kind = measured_peak_hbm()
    mine = torch.tensor([phase[3], phase[5], p2g_b, g2p_b], dtype=torch.float64, device=dev)
    allr = [torch.zeros(4, dtype=torch.float64, device=dev) for _ in range(ws)]
    dist.all_gather(allr, mine)
    rows = [r.cpu().numpy() for r in allr]
    worst = max(rows, key=lambda r: r[0] + r[1])
    dom_p2g = worst[0] >= worst[1]
    dom_b, dom_ms = (worst[2], worst[0]) if dom_p2g else (worst[3], worst[1])
    achieved = dom_b / (dom_ms * 1e-3) / 1e9
    # e2e: each step the rank's state goes host -> device -> host through the ABI
    e2e_steps = max(1, args.e2e_steps)
    dist.barrier()
    L.ckg_timer_mark(rk.ctx, 2)
    hb = hd = 0
    for _ in range(e2e_steps):
        host = rk.particles()
        hd += host.nbytes
        L.ckg_upload(rk.ctx, abi.ptr(host), len(host))
        hb += host.nbytes
        tr.step(rk, dt)
    L.ckg_timer_mark(rk.ctx, 3)
    L.ckg_timer_elapsed(rk.ctx, 2, 3, C.byref(el))
    t = torch.tensor([el.value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if args.precision == 8 else "f32",
            "data": "synthetic",
            "config": bench_config(args, cells, n_total, dt),
            "parallelism": f"x-slab decomposition over {ws} GPUs (NCCL halo reduce / velocity broadcast, "
                           f"ordered migration), {args.scaling} scaling",
            "slab_bounds": list(map(int, bounds)), "slab_bounds_final": list(map(int, rk.bounds)),
            "rebalance_every": args.rebalance_every,
            "phase_ms_rank0": dict(zip(abi.PHASE_NAMES, phase.tolist())),
            "e2e": {"value": n_total * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": hb // e2e_steps, "d2h_bytes_per_step": hd // e2e_steps,
                    "steps": e2e_steps, "path": "per rank: ckg_download + ckg_upload + slab substep"},
            "gpu_launches": launches, "clocks": clocks,
            "roofline": {"bound": "hbm", "kernel": "p2g_kernel" if dom_p2g else "g2p_kernel",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "algorithmic_bytes": dom_b,
                         "avg_ms": dom_ms, "rank": "slowest rank (max P2G + G2P time)"},
            "cpu_baseline": None,  # measured at N=1 only (the reference arm runs this config)
        }
        print(json.dumps(line), flush=True)
    rk.close()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    ws, rank, local = dist_env()
    if ws > 1 or args.force_slab:
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29577")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        run_slab(args, ws, rank, local)
        return
    dist = None
    import torch

    from paper_2412_10399_b200._lib import lib
    from paper_2412_10399_b200.api import Simulation

    L = lib()
    prec = args.precision
    cells = workload_cells(args, 1)
    cfg = bench_scene(args, cells)
    host = seed_particles(cfg, prec)
    n = len(host)
    sim = Simulation(cfg, precision=prec, device=local, particles=host, fused=True if args.fused else None)
    fused = sim.fused()
    ctx = sim._ctx
    dt = sim.cfl_dt(1.0)
    out = abi.StepOut()

    def step_once():
        rc = L.ckg_step(ctx, dt, C.byref(out))
        if rc != 0:
            buf = C.create_string_buffer(256)
            L.ckg_last_error_message(ctx, buf, 256)
            raise RuntimeError(f"ckg_step failed: {buf.value.decode()}")

    for _ in range(args.warmup):
        step_once()
    # phase shares from one steady-state step (device events on the library stream)
    step_once()
    phase_ms = list(out.phase_ms)
    nblocks = int(out.active_blocks)
    launches_per_step = int(out.kernel_launches)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    time.sleep(0.3)
    L.ckg_timer_mark(ctx, 0)
    p2g_ms, g2p_ms = [], []
    phase_acc = [0.0] * 6
    sort_kinds = []
    total_launch = 0
    for _ in range(args.steps):
        step_once()
        p2g_ms.append(out.phase_ms[3])
        g2p_ms.append(out.phase_ms[5])
        for k in range(6):
            phase_acc[k] += out.phase_ms[k] / args.steps
        sort_kinds.append(int(out.sort_kind))
        total_launch += int(out.kernel_launches)
    L.ckg_timer_mark(ctx, 1)
    el_ms = C.c_double()
    L.ckg_timer_elapsed(ctx, 0, 1, C.byref(el_ms))
    clocks = sampler.stop()
    barrier()
    t_ms = el_ms.value
    if dist is not None:
        tt = torch.tensor([t_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = n * ws * args.steps / (t_ms * 1e-3)

    # e2e: the same substep through the C-ABI with HOST buffers: each step
    # uploads the full Particle<T> AoS from pinned host memory, steps, and
    # downloads the new state into the same buffer (the next step's input: a
    # host-resident simulation).  `chains` such simulations (same scene, own
    # context each) run in their own host threads, so one chain's upload can
    # overlap another's download (PCIe is full duplex) and substep.
    nbytes = n * abi.particle_dtype(prec).itemsize
    e2e_steps = max(1, args.e2e_steps)
    chains = max(1, args.e2e_chains)
    ctxs = [ctx]
    extra = []
    for _ in range(chains - 1):
        extra.append(Simulation(cfg, precision=prec, device=local, particles=host,
                                fused=True if args.fused else None))
        ctxs.append(extra[-1]._ctx)
    bufs = []
    for k in range(chains):
        b = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(abi.particle_dtype(prec))
        b[:] = host
        bufs.append(b)
    errors = []

    def chain(k, steps):
        o = abi.StepOut()
        try:
            for _ in range(steps):
                assert L.ckg_upload(ctxs[k], abi.ptr(bufs[k]), n) == 0
                assert L.ckg_step(ctxs[k], dt, C.byref(o)) == 0
                assert L.ckg_download(ctxs[k], abi.ptr(bufs[k]), n) == 0
        except Exception as e:  # surfaced below, never swallowed
            errors.append(e)

    def run_chains(steps):
        ts = [threading.Thread(target=chain, args=(k, steps)) for k in range(chains)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    def timed(nch, steps):
        """Wall time of `steps` substeps on each of the first `nch` chains."""
        nonlocal chains
        saved, chains = chains, nch
        try:
            run_chains(1)  # untimed warm-up (first pinned transfers, allocator)
            barrier()
            w = run_chains(steps)
        finally:
            chains = saved
        if errors:
            raise errors[0]
        ms = w * 1e3
        if dist is not None:
            tt = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return n * nch * ws * steps / (ms * 1e-3)

    # headline: ONE drop-in simulation, host-resident state
    e2e_val = timed(1, e2e_steps)
    # secondary: `chains` concurrent simulations (one's upload overlaps
    # another's download and substep)
    e2e_multi = timed(chains, e2e_steps) if chains > 1 else None
    for s in extra:
        s.close()

    # roofline of the dominant kernel (device events around each launch)
    p2g_bytes, g2p_bytes = algorithmic_bytes(n, nblocks, args.scheme, prec)
    p2g_avg = float(np.mean(p2g_ms))
    g2p_avg = float(np.mean(g2p_ms))
    peak, peak_kind = measured_peak_hbm()
    if fused:
        # one kernel: G2P of this substep + P2G of the next (its P2G phase
        # slot only promotes the pending scatter's status)
        dom, dom_bytes, dom_ms = "g2p2g_kernel", p2g_bytes + g2p_bytes, g2p_avg
    elif p2g_avg >= g2p_avg:
        dom, dom_bytes, dom_ms = "p2g_kernel", p2g_bytes, p2g_avg
    else:
        dom, dom_bytes, dom_ms = "g2p_kernel", g2p_bytes, g2p_avg
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    flops = {}
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            traffic = tj.get(dom)
            flops = tj.get("fp64_flop_per_launch", {})
        except Exception:
            traffic = None
    # the FP64 pipe as the second ceiling: ncu's FP64 op count of
    # the same launch (bench scene only) over the live kernel time, against the
    # measured DFMA peak (tools/fp64_peak.cu -> profiles/fp64_peak.json)
    roof64 = None
    try:
        peak64 = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_fma_tflops"]
        if prec == 8 and cells == 108 and args.scheme == "apic" and args.model == "fixed_corotated" and not fused \
                and "p2g_kernel" in flops:
            f_p2g, f_g2p = flops["p2g_kernel"], flops["g2p_kernel"]
            roof64 = {"bound": "fp64", "unit": "TFLOP/s", "peak": peak64, "peak_kind": "measured (DFMA loop)",
                      "p2g": f_p2g / (p2g_avg * 1e-3) / 1e12, "g2p": f_g2p / (g2p_avg * 1e-3) / 1e12,
                      "p2g_frac": f_p2g / (p2g_avg * 1e-3) / 1e12 / peak64,
                      "g2p_frac": f_g2p / (g2p_avg * 1e-3) / 1e12 / peak64,
                      "flop_source": flops.get("source")}
    except Exception:
        roof64 = None

    single = None
    if ws == 1 and prec == 8 and not args.no_single:
        sim.close()
        try:
            single = single_precision_rate(args, cfg, local)
            # the same algorithmic-bytes roofline for the FP32 transfer kernels
            sb = algorithmic_bytes(n, nblocks, args.scheme, 4)
            sp2g, sg2p = single["phase_ms"]["p2g"], single["phase_ms"]["g2p"]
            single["p2g_g2p"] = {"p2g_gbs": None if single["fused"] else sb[0] / (sp2g * 1e-3) / 1e9,
                                 "g2p_gbs": None if single["fused"] else sb[1] / (sg2p * 1e-3) / 1e9,
                                 "combined_gbs": (sb[0] + sb[1]) / ((sp2g + sg2p) * 1e-3) / 1e9,
                                 "combined_frac": (sb[0] + sb[1]) / ((sp2g + sg2p) * 1e-3) / 1e9 / peak}
        except Exception as e:  # reported, never silently substituted
            single = {"value": None, "error": str(e)}
    if rank == 0:
        cb = None
        if not args.no_cpu_baseline and ws == 1:
            try:
                cb = cpu_baseline(args, os.cpu_count() or 1)
            except Exception as e:  # reported, never silently substituted
                cb = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                      "sample": f"unavailable: {e}"}
        ms_step = t_ms / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64" if prec == 8 else "f32", "data": "synthetic",
            "config": bench_config(args, cells, n, dt, nblocks),
            "parallelism": "single GPU" if ws == 1 else f"{ws} independent replicas (weak)",
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "frac_vs_spec_8tbs": achieved / 8000.0,
                         "traffic": traffic, "algorithmic_bytes": dom_bytes, "avg_ms": dom_ms},
            "roofline_fp64": roof64,
            "transfer_path": "fused G2P2G kernel (G2P of substep n + P2G of n+1)" if fused else
                             "separate P2G and G2P kernels",
            "p2g_g2p": {"p2g_ms": p2g_avg, "g2p_ms": g2p_avg,
                        "p2g_gbs": None if fused else p2g_bytes / (p2g_avg * 1e-3) / 1e9,
                        "g2p_gbs": None if fused else g2p_bytes / (g2p_avg * 1e-3) / 1e9,
                        "combined_gbs": (p2g_bytes + g2p_bytes) / ((p2g_avg + g2p_avg) * 1e-3) / 1e9,
                        "combined_frac": (p2g_bytes + g2p_bytes) / ((p2g_avg + g2p_avg) * 1e-3) / 1e9 / peak},
            "phase_ms": dict(zip(abi.PHASE_NAMES, phase_acc)),
            "sort_kinds": {"full_radix": sort_kinds.count(0), "identity": sort_kinds.count(1),
                           "incremental": sort_kinds.count(2)},
            "cpu_baseline": cb,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "steps": e2e_steps, "chains": 1,
                    "path": "one drop-in simulation: per step ckg_upload(pinned Particle<T> AoS) + ckg_step + "
                            "ckg_download into the same buffer (the next step's input); wall clock"},
            "e2e_multi_chain": None if e2e_multi is None else {
                "value": e2e_multi, "unit": UNIT, "chains": chains, "steps": e2e_steps,
                "h2d_bytes_per_step": nbytes * chains, "d2h_bytes_per_step": nbytes * chains,
                "path": "`chains` independent host-resident simulations of the same scene stepped concurrently "
                        "(one host thread each); aggregate particle-substeps/s"},
            "gpu_launches": total_launch,
            "launches_per_step": launches_per_step,
            "clocks": clocks,
            "single_precision": single,
        }
        print(json.dumps(line), flush=True)
    if single is None:
        sim.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
