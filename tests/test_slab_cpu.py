"""Multi-rank host logic of the x-slab decomposition on CPU (gloo,
world_size 2 and 3): slab partitioning, and the transport's exchange
semantics for every request type the substep issues."""
import os
import socket

import numpy as np
import pytest

from paper_2412_10399_b200.scene import block_scene, seed_particles
from paper_2412_10399_b200.slab import (AllReduceMax, Counts, DistTransport, Join, Neighbor, Scalars, block_x_of,
                                        partition_planes, split_particles)


def test_partition_balances_and_covers():
    counts = np.array([0, 0, 5, 100, 100, 100, 100, 50, 0, 0])
    for world in (1, 2, 3, 4):
        b = partition_planes(counts, world)
        assert b[0] == 0 and b[-1] == len(counts) and all(b[i] < b[i + 1] for i in range(world))
        loads = [counts[b[i]:b[i + 1]].sum() for i in range(world)]
        assert max(loads) - min(loads) <= 2 * counts.max()


def test_split_preserves_global_stable_order():
    cfg = block_scene(16, resolution=64)
    p = seed_particles(cfg)
    p = p[np.random.default_rng(0).permutation(len(p))]
    bounds, parts = split_particles(p, cfg, 3)
    cat = np.concatenate(parts)
    # concatenation of the slabs == the global stable sort by block key
    D = 64 // 4 + 2
    c = np.clip(np.floor(p["x"] * 64.0 + 0.25).astype(np.int64) >> 2, 0, D - 1)
    key = (c[:, 0] * D + c[:, 1]) * D + c[:, 2]
    assert cat.tobytes() == p[np.argsort(key, kind="stable")].tobytes()
    for r, part in enumerate(parts):
        bx = block_x_of(part, cfg)
        assert np.all((bx >= bounds[r]) & (bx < bounds[r + 1]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = DistTransport(dist, rank, world, torch.device("cpu"))
    res = {}
    # MAX all-reduce of footprint flags
    flags = torch.zeros(16, dtype=torch.int32)
    flags[rank] = 1
    tr.handle(AllReduceMax(flags))
    res["flags"] = flags.tolist()
    # neighbour exchange: ghost planes to owners (sizes differ per side)
    sl = torch.full((rank + 1,), float(10 * rank + 1)) if rank > 0 else None
    sr = torch.full((rank + 2,), float(10 * rank + 2)) if rank < world - 1 else None
    rl = torch.zeros(rank - 1 + 2) if rank > 0 else None          # left neighbour sends (r-1)+2
    rr = torch.zeros(rank + 1 + 1) if rank < world - 1 else None  # right neighbour sends (r+1)+1
    tr.handle(Neighbor(sl, sr, rl, rr))
    res["rl"] = None if rl is None else rl.tolist()
    res["rr"] = None if rr is None else rr.tolist()
    # the same exchange as an overlap request completed by Join (the P2G
    # halo's protocol: in flight while the interior planes scatter)
    rl2 = torch.zeros_like(rl) if rl is not None else None
    rr2 = torch.zeros_like(rr) if rr is not None else None
    tr.handle(Neighbor(sl, sr, rl2, rr2, overlap=True))
    tr.handle(Join())
    res["overlap_same"] = all(a is None and b is None or (a is not None and b is not None and a.tolist() == b.tolist())
                              for a, b in ((rl, rl2), (rr, rr2)))
    got = [None, None]
    tr.handle(Counts(100 + rank, 200 + rank, got))
    res["counts"] = got
    out = [None]
    tr.handle(Scalars(np.array([float(rank), -float(rank + 1), 0.0]), out))
    res["scalars"] = out[0].tolist()
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_transport_semantics_gloo(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        d = res[r]
        assert d["flags"][:world] == [1] * world
        if r > 0:
            assert d["rl"] == [float(10 * (r - 1) + 2)] * (r - 1 + 2)
            assert d["counts"][0] == 200 + (r - 1)
        else:
            assert d["rl"] is None and d["counts"][0] == 0
        if r < world - 1:
            assert d["rr"] == [float(10 * (r + 1) + 1)] * (r + 2)
            assert d["counts"][1] == 100 + (r + 1)
        else:
            assert d["rr"] is None and d["counts"][1] == 0
        assert d["scalars"] == [float(world - 1), -1.0, 0.0]
        assert d["overlap_same"]


C4_SMALL = {"name": "c4_small", "resolution": 64, "scheme": "apic", "gravity": [0, -0.1, 0],
            "materials": [{"model": "drucker_prager", "density": 1400.0, "E": 10000.0, "nu": 0.4,
                           "friction_angle_deg": 30.0},
                          {"model": "fixed_corotated", "density": 1000.0, "E": 10000000.0, "nu": 0.2}],
            "bodies": [{"shape": {"kind": "box", "lo": [0.40625, 0.0625, 0.39453125],
                                  "hi": [0.6171875, 0.2734375, 0.60546875]}, "material": 0, "ppc": 8},
                       {"shape": {"kind": "sphere", "center": [0.30625, 0.16796875, 0.5], "radius": 0.0625},
                        "material": 1, "ppc": 8, "velocity": [10.0, 0, 0]},
                       {"shape": {"kind": "cylinder", "center": [0.7, 0.2, 0.5], "radius": 0.05,
                                  "half_length": 0.08, "axis": 1}, "material": 1, "ppc": 27}],
            "boundaries": [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625, 1], "normal": [0, 1, 0]}]}


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("precision", [8, 4])
def test_rank_local_seeding_multibody(world, precision):
    """Rank-local seeding of a multi-body scene (sandcastle-like: DP box, fast
    FC ball, ppc-27 cylinder): each rank's part, stably sorted by block key,
    is bit-identical to its slab of the globally seeded and sorted set, and
    mass_eps / vmax are the global ones."""
    from paper_2412_10399_b200.scene import SceneConfig, mass_epsilon, seed_particles
    from paper_2412_10399_b200.slab import rank_local_particles, split_particles

    cfg = SceneConfig.from_json(C4_SMALL, precision)
    full = seed_particles(cfg, precision)
    bounds_ref, parts_ref = split_particles(full, cfg, world, precision)
    T = np.float64 if precision == 8 else np.float32
    D = cfg.resolution // 4 + 2
    inv_dx = T(1) / cfg.dx(precision)
    for r in range(world):
        bounds, part, me, vmax = rank_local_particles(cfg, world, r, precision)
        assert bounds == bounds_ref
        c = np.clip(np.floor(part["x"].astype(T) * inv_dx + T(0.25)).astype(np.int64) >> 2, 0, D - 1)
        key = (c[:, 0] * D + c[:, 1]) * D + c[:, 2]
        got = part[np.argsort(key, kind="stable")]
        assert got.tobytes() == parts_ref[r].tobytes(), r
        assert me == mass_epsilon(full, precision)
        assert vmax == pytest.approx(10.0)
