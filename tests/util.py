"""Shared test helpers: scene builders and tolerant comparisons."""
import numpy as np

from paper_2412_10399_b200.scene import SceneConfig


def close(a, b, tol):
    """|a-b| <= tol*max(1,|a|,|b|) — test_helpers.hpp:18-21."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return np.abs(a - b) <= tol * scale


def max_rel(a, b, floor=1.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(floor, np.maximum(np.abs(a), np.abs(b)))
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def small_scene(scheme="apic", model="fixed_corotated", res=32, bc="sticky", gravity=(0, -9.8, 0),
                lo=(0.34375, 0.3125, 0.34375), hi=(0.59375, 0.5625, 0.59375), velocity=(0.0, 0.0, 0.0),
                E=1e5, nu=0.4, density=1000.0, extra_mats=(), ppc=8, shape="box", omega=(0.0, 0.0, 0.0)):
    mat = {"model": model, "density": density}
    if model == "j_fluid":
        mat.update({"bulk": 1e4, "gamma": 7.0, "viscosity": 0.1})
    else:
        mat.update({"E": E, "nu": nu})
        if model == "drucker_prager":
            mat["friction_angle_deg"] = 30.0
    if shape == "box":
        sh = {"kind": "box", "lo": list(lo), "hi": list(hi)}
    else:
        c = [(lo[a] + hi[a]) / 2 for a in range(3)]
        sh = {"kind": "sphere", "center": c, "radius": (hi[0] - lo[0]) / 2}
    obj = {"name": "t", "resolution": res, "scheme": scheme, "gravity": list(gravity),
           "materials": [mat] + list(extra_mats),
           "bodies": [{"shape": sh, "material": 0, "ppc": ppc, "velocity": list(velocity),
                       "omega": list(omega)}],
           "boundaries": []}
    if bc == "sticky":
        obj["boundaries"] = [{"kind": "sticky", "lo": [0, 0, 0], "hi": [1, 0.0625 * 4, 1]}]
    elif bc == "separate":
        obj["boundaries"] = [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, 0.0625 * 4, 1], "normal": [0, 1, 0]}]
    elif bc == "slip":
        obj["boundaries"] = [{"kind": "slip", "lo": [0, 0, 0], "hi": [1, 0.0625 * 4, 1], "normal": [0, 1, 0]}]
    return SceneConfig.from_json(obj)


def perturb(p, seed=0, fscale=0.05, vscale=0.3, bscale=0.5, xscale=0.3, dx=1.0 / 32):
    """Randomise a seeded state so every term of the transfer is exercised."""
    rng = np.random.default_rng(seed)
    q = p.copy()
    n = len(q)
    T = q["x"].dtype.type
    q["x"] = q["x"] + (rng.uniform(-xscale, xscale, (n, 3)) * dx).astype(T)
    q["v"] = rng.uniform(-vscale, vscale, (n, 3)).astype(T)
    q["F"] = (np.eye(3) + rng.uniform(-fscale, fscale, (n, 3, 3))).astype(T)
    q["B"] = (rng.uniform(-bscale, bscale, (n, 3, 3)) * dx * dx).astype(T)
    return q
