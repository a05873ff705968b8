"""Helpers for the -m gpu parity tests (the device path is always the C-ABI)."""
import numpy as np

from paper_2412_10399_b200 import abi
from paper_2412_10399_b200.api import Simulation


def tag_volumes(p):
    """Make volume0 unique per particle (tiny relative spread) so particles can
    be matched across independently sorted runs; physics stays well-posed and
    every engine sees the same inputs."""
    q = p.copy()
    T = q["volume0"].dtype.type
    q["volume0"] = (q["volume0"] * (T(1) + np.arange(len(q), dtype=q["volume0"].dtype) * T(2.0 ** -36))).astype(T)
    return q


def match_by_tag(a, b):
    ia = np.argsort(a["volume0"], kind="stable")
    ib = np.argsort(b["volume0"], kind="stable")
    assert np.array_equal(a["volume0"][ia], b["volume0"][ib]), "particle sets differ"
    return a[ia], b[ib]


def field_rel(a, b, name, floor=1e-300):
    x = np.asarray(a[name], dtype=np.float64).reshape(len(a), -1)
    y = np.asarray(b[name], dtype=np.float64).reshape(len(b), -1)
    scale = max(np.max(np.abs(y)) if y.size else 0.0, floor)
    return float(np.max(np.abs(x - y)) / scale) if x.size else 0.0


def gpu_sim(cfg, particles, precision=8, fused=None):
    return Simulation(cfg, precision=precision, particles=particles, fused=fused)


def nodes_by_coord(coords, nodes):
    return {tuple(c): nodes[i] for i, c in enumerate(coords)}
