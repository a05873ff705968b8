"""Host-side mirror of the reference's scene / config / material API.

The reference keeps these on the host (proj/include/ckmpm/scene.hpp,
material.hpp, io.hpp); so does this build.  Everything here is plain host
logic that feeds the device through the C-ABI:

* ``SceneConfig.from_json`` reads the reference's strict JSON scene schema
  (io.hpp:242-315) with its pinned defaults;
* ``finalize_material`` restates material.hpp:52-88 (Lame parameters, DP
  alpha) with the reference's operation order, in the config's precision;
* ``seed_particles`` restates scene.hpp:78-131, :204-230 (deterministic
  lattice seeding, ppc 8/27; jittered ppc 16 via mt19937_64), vectorised;
* ``mass_epsilon`` restates Simulation::compute_mass_epsilon
  (simulation.hpp:227-232).

Seeding is pinned bit-exact against the reference sampler in
tests/test_scene.py.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi


class ConfigError(RuntimeError):
    """Reference ConfigError (errors.hpp:10-12) -> exit code 2."""


class NumericalError(RuntimeError):
    """Reference NumericalError (errors.hpp:14-16) -> exit code 3."""


class IoError(RuntimeError):
    """Reference IoError (errors.hpp:18-20) -> exit code 4."""


class OutOfDomainError(NumericalError):
    """Reference OutOfDomainError (errors.hpp:23-27), carries particle_index."""

    def __init__(self, particle_index: int, what: str):
        super().__init__(what)
        self.particle_index = particle_index


class InvertedElementError(NumericalError):
    """Reference InvertedElementError (errors.hpp:30-32)."""


class DeviceError(RuntimeError):
    """CUDA/runtime failure of the B200 backend (no reference equivalent)."""


_libm = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
_libm.sinf.argtypes = [ctypes.c_float]
_libm.sinf.restype = ctypes.c_float


def _T(precision: int):
    return np.float64 if precision == 8 else np.float32


def _sin(x, precision):
    if precision == 8:
        return math.sin(float(x))
    return np.float32(_libm.sinf(float(x)))


@dataclass
class Material:
    model: str = "fixed_corotated"
    density: float = 0.0
    E: float = 0.0
    nu: float = 0.0
    bulk: float = 0.0
    gamma: float = 0.0
    viscosity: float = 0.0
    friction_angle_deg: float = 0.0
    mu: float = 0.0
    lam: float = 0.0
    dp_alpha: float = 0.0

    @property
    def is_fluid(self) -> bool:
        return self.model == "j_fluid"


def finalize_material(m: Material, precision: int = 8) -> Material:
    """material.hpp:52-88 (lame_from_E_nu :24-31, dp_alpha_from_friction_deg :52-57)."""
    T = _T(precision)
    if not (T(m.density) > 0):
        raise ConfigError("density: must be > 0")
    if m.model in ("fixed_corotated", "drucker_prager"):
        E, nu = T(m.E), T(m.nu)
        if not (E > 0):
            raise ConfigError("E: must be > 0")
        if not (nu >= 0 and nu < T(0.5)):
            raise ConfigError("nu: must satisfy 0 <= nu < 0.5")
        m.mu = float(E / (T(2) * (T(1) + nu)))
        m.lam = float(E * nu / ((T(1) + nu) * (T(1) - T(2) * nu)))
        if m.model == "drucker_prager":
            deg = T(m.friction_angle_deg)
            if not (deg > 0 and deg < 90):
                raise ConfigError("friction_angle: must lie in (0, 90) degrees")
            phi = deg * T(math.pi) / T(180)
            s = T(_sin(phi, precision))
            m.dp_alpha = float(T(np.sqrt(T(2) / T(3))) * T(2) * s / (T(3) - s))
    elif m.model == "j_fluid":
        if not (T(m.bulk) > 0):
            raise ConfigError("B: must be > 0")
        if not (T(m.gamma) > 1):
            raise ConfigError("gamma: must be > 1")
        if not (T(m.viscosity) >= 0):
            raise ConfigError("viscosity: must be >= 0")
    elif m.model in ("nacc", "von_mises"):
        raise ConfigError(f"material '{m.model}' is a reserved tag and not implemented")
    else:
        raise ConfigError(f"unknown material model '{m.model}'")
    return m


@dataclass
class Shape:
    kind: str = "sphere"
    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 0.0
    inner_radius: float = 0.0
    half_length: float = 0.0
    axis: int = 1
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (0.0, 0.0, 0.0)


@dataclass
class Body:
    shape: Shape
    material: int = 0
    ppc: int = 8
    seed: int = 0
    velocity: tuple = (0.0, 0.0, 0.0)
    shear_slope: float = 0.0
    omega: tuple = (0.0, 0.0, 0.0)


@dataclass
class Boundary:
    kind: str = "sticky"
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (0.0, 0.0, 0.0)
    normal: tuple = (0.0, 0.0, 0.0)
    velocity: tuple = (0.0, 0.0, 0.0)
    omega: tuple = (0.0, 0.0, 0.0)
    center: tuple = (0.0, 0.0, 0.0)


@dataclass
class SceneConfig:
    """SimConfig<T> (scene.hpp:159-182) with the reference defaults."""
    name: str = "scene"
    resolution: int = 64
    extent: float = 1.0
    kernel: str = "compact"
    scheme: str = "apic"
    gravity: tuple = (0.0, 0.0, 0.0)
    cfl: float = 0.5
    frame_dt: float = 1.0 / 60.0
    frames: int = 1
    max_dt: float = 0.0
    deterministic: bool = False
    threads: int = 0
    clamp_singular: bool = False
    clamp_floor: float = 0.05
    max_substeps_per_frame: int = 1000000
    materials: List[Material] = field(default_factory=list)
    bodies: List[Body] = field(default_factory=list)
    boundaries: List[Boundary] = field(default_factory=list)

    def dx(self, precision: int = 8):
        T = _T(precision)
        return T(self.extent) / T(self.resolution)  # scene.hpp:181

    def validate(self) -> None:
        """validate_config (scene.hpp:184-200)."""
        if self.resolution < 8:
            raise ConfigError("resolution: must be at least 8")
        if not (self.extent > 0):
            raise ConfigError("extent: must be positive")
        if not (self.cfl > 0) or self.cfl > 1:
            raise ConfigError("cfl: must be in (0, 1]")
        if not (self.frame_dt > 0):
            raise ConfigError("frame_dt: must be positive")
        if self.frames < 0:
            raise ConfigError("frames: must be non-negative")
        if not self.materials:
            raise ConfigError("materials: at least one required")
        if not self.bodies:
            raise ConfigError("bodies: at least one required")
        if self.kernel == "quadratic" and self.scheme == "mls":
            raise ConfigError("scheme: mls requires the compact kernel")  # scene.hpp:193-194
        for b in self.bodies:
            if b.material >= len(self.materials):
                raise ConfigError("bodies: material index out of range")

    @staticmethod
    def from_json(obj, precision: int = 8) -> "SceneConfig":
        """config_from_json (io.hpp:242-315): strict field set, pinned defaults."""
        if isinstance(obj, str):
            obj = json.loads(obj)
        allowed = {"name", "resolution", "extent", "kernel", "scheme", "gravity", "cfl", "frame_dt",
                   "frames", "max_dt", "deterministic", "threads", "clamp_singular", "clamp_floor",
                   "max_substeps_per_frame", "materials", "bodies", "boundaries", "output"}
        for k in obj:
            if k not in allowed:
                raise ConfigError(f"config.{k}: unknown field")
        c = SceneConfig()
        c.name = obj.get("name", "scene")
        if "resolution" not in obj:
            raise ConfigError("config.resolution: required")
        c.resolution = int(obj["resolution"])
        c.extent = float(obj.get("extent", 1.0))
        c.kernel = obj.get("kernel", "compact")
        if c.kernel not in ("compact", "quadratic"):
            raise ConfigError("config.kernel: expected 'compact' or 'quadratic'")  # io.hpp:255-261
        c.scheme = obj.get("scheme", "apic")
        if c.scheme not in abi.SCHEME_NAMES:
            raise ConfigError("config.scheme: expected 'pic', 'apic' or 'mls'")
        c.gravity = tuple(float(v) for v in obj.get("gravity", (0.0, 0.0, 0.0)))
        c.cfl = float(obj.get("cfl", 0.5))
        c.frame_dt = float(obj.get("frame_dt", 1.0 / 60.0))
        c.frames = int(obj.get("frames", 1))
        c.max_dt = float(obj.get("max_dt", 0.0))
        c.deterministic = bool(obj.get("deterministic", False))
        c.threads = int(obj.get("threads", 0))
        c.clamp_singular = bool(obj.get("clamp_singular", False))
        c.clamp_floor = float(obj.get("clamp_floor", 0.05))
        c.max_substeps_per_frame = int(obj.get("max_substeps_per_frame", 1000000))
        for i, m in enumerate(obj["materials"]):
            mat = Material(model=m["model"], density=float(m["density"]))
            if mat.model == "j_fluid":
                mat.bulk, mat.gamma = float(m["bulk"]), float(m["gamma"])
                mat.viscosity = float(m.get("viscosity", 0.0))
            else:
                mat.E, mat.nu = float(m.get("E", 0.0)), float(m.get("nu", 0.0))
                if mat.model == "drucker_prager":
                    mat.friction_angle_deg = float(m["friction_angle_deg"])
            try:
                finalize_material(mat, precision)
            except ConfigError as e:
                raise ConfigError(f"materials[{i}].{e}") from None
            c.materials.append(mat)
        for b in obj["bodies"]:
            s = b["shape"]
            sh = Shape(kind=s["kind"])
            if sh.kind == "sphere":
                sh.center, sh.radius = tuple(s["center"]), float(s["radius"])
            elif sh.kind == "box":
                sh.lo, sh.hi = tuple(s["lo"]), tuple(s["hi"])
            elif sh.kind == "cylinder":
                sh.center, sh.radius = tuple(s["center"]), float(s["radius"])
                sh.inner_radius = float(s.get("inner_radius", 0.0))
                sh.half_length = float(s["half_length"])
                sh.axis = int(s.get("axis", 1))
            else:
                raise ConfigError(f"unknown shape '{sh.kind}'")
            c.bodies.append(Body(shape=sh, material=int(b["material"]), ppc=int(b.get("ppc", 8)),
                                 seed=int(b.get("seed", 0)),
                                 velocity=tuple(b.get("velocity", (0.0, 0.0, 0.0))),
                                 shear_slope=float(b.get("shear_slope", 0.0)),
                                 omega=tuple(b.get("omega", (0.0, 0.0, 0.0)))))
        for bc in obj.get("boundaries", []):
            B = Boundary(kind=bc["kind"], lo=tuple(bc["lo"]), hi=tuple(bc["hi"]))
            if B.kind != "sticky":
                nrm = np.array(bc["normal"], dtype=np.float64)
                T = _T(precision)
                nrm = nrm.astype(T)
                n = T(np.sqrt(T(nrm[0] * nrm[0] + nrm[1] * nrm[1]) + nrm[2] * nrm[2]))
                if not (n > 0):
                    raise ConfigError("normal: must be nonzero")
                inv = T(1) / n
                B.normal = tuple(float(T(v) * inv) for v in nrm)
            else:
                B.velocity = tuple(bc.get("velocity", (0.0, 0.0, 0.0)))
                B.omega = tuple(bc.get("omega", (0.0, 0.0, 0.0)))
                B.center = tuple(bc.get("center", (0.0, 0.0, 0.0)))
            c.boundaries.append(B)
        c.validate()
        return c


# ------------------------------------------------------------------ seeding

class _MT19937_64:
    """std::mt19937_64 (for the jittered ppc=16 sampler, scene.hpp:112-125)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def next(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def uniform(self) -> float:
        # libstdc++ generate_canonical<double, 53> with a 64-bit engine.
        r = self.next() / 18446744073709551616.0
        return r if r < 1.0 else math.nextafter(1.0, 0.0)

    def uniform_f32(self):
        """libstdc++ generate_canonical<float, 24> with a 64-bit engine: the
        draw is rounded to float ONCE (uint64 -> float, ties to even), divided
        in float by float(2^64), and a result >= 1 is clamped to
        nextafter(1.0f, 0) (uniform_real_distribution<float>(0, 1))."""
        r = _u64_to_f32(self.next()) / np.float32(18446744073709551616.0)
        return r if r < np.float32(1.0) else np.nextafter(np.float32(1.0), np.float32(0.0))


def _u64_to_f32(n: int) -> np.float32:
    """Correctly rounded uint64 -> float32 (one rounding, ties to even; a
    conversion through float64 could round twice)."""
    b = n.bit_length()
    if b <= 24:
        return np.float32(n)
    shift = b - 24
    q = n >> shift
    rem = n & ((1 << shift) - 1)
    half = 1 << (shift - 1)
    if rem > half or (rem == half and (q & 1)):
        q += 1
    return np.float32(q) * np.float32(2.0 ** shift)  # exact: q <= 2^24, power-of-two scale


def _shape_mask(shape: Shape, X, Y, Z, T):
    if shape.kind == "sphere":
        c = [T(v) for v in shape.center]
        dx_, dy_, dz_ = X - c[0], Y - c[1], Z - c[2]
        r = T(shape.radius)
        return (dx_ * dx_ + dy_ * dy_) + dz_ * dz_ < r * r
    if shape.kind == "box":
        lo = [T(v) for v in shape.lo]
        hi = [T(v) for v in shape.hi]
        return (X >= lo[0]) & (X < hi[0]) & (Y >= lo[1]) & (Y < hi[1]) & (Z >= lo[2]) & (Z < hi[2])
    if shape.kind == "cylinder":
        c = [T(v) for v in shape.center]
        d = [X - c[0], Y - c[1], Z - c[2]]
        along = d[shape.axis]
        ok = np.abs(along) < T(shape.half_length)
        d[shape.axis] = np.zeros_like(along)
        r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
        ok &= r2 < T(shape.radius) * T(shape.radius)
        ok &= r2 >= T(shape.inner_radius) * T(shape.inner_radius)
        return ok
    raise ConfigError(f"unknown shape '{shape.kind}'")


def _aabb(shape: Shape, T):
    if shape.kind == "sphere":
        c = [T(v) for v in shape.center]
        r = T(shape.radius)
        return [c[a] - r for a in range(3)], [c[a] + r for a in range(3)]
    if shape.kind == "box":
        return [T(v) for v in shape.lo], [T(v) for v in shape.hi]
    c = [T(v) for v in shape.center]
    ext = [T(shape.radius)] * 3
    ext[shape.axis] = T(shape.half_length)
    return [c[a] - ext[a] for a in range(3)], [c[a] + ext[a] for a in range(3)]


def sample_shape(shape: Shape, dx, ppc: int, seed: int = 0, precision: int = 8,
                 i_range: Optional[tuple] = None) -> np.ndarray:
    """sample_shape (scene.hpp:78-131): (n, 3) positions in emission order.

    i_range = (lo, hi): only the lattice cells with lo <= i <= hi (the outer,
    x loop), i.e. exactly that part of the emission order (ppc 8 / 27; the
    jittered ppc 16 draws its random stream over every cell and ignores it)."""
    T = _T(precision)
    dx = T(dx)
    if not (dx > 0):
        raise ConfigError("sample_shape: dx must be positive")
    blo, bhi = _aabb(shape, T)
    i0, j0, k0 = (int(math.floor(T(blo[a]) / dx)) - 1 for a in range(3))
    i1, j1, k1 = (int(math.ceil(T(bhi[a]) / dx)) + 1 for a in range(3))
    if ppc in (8, 27):
        nsub = 2 if ppc == 8 else 3
        offs = np.array([T(2 * s + 1) / T(2 * nsub) for s in range(nsub)], dtype=T)
        ii = np.arange(i0 if i_range is None else max(i0, i_range[0]),
                       (i1 if i_range is None else min(i1, i_range[1])) + 1)
        jj = np.arange(j0, j1 + 1)
        kk = np.arange(k0, k1 + 1)
        # loop order i, j, k, a, b, c (scene.hpp:90-101)
        I, J, K, A, B, Cc = np.meshgrid(ii, jj, kk, np.arange(nsub), np.arange(nsub), np.arange(nsub),
                                        indexing="ij")
        X = (I.astype(T) + offs[A]) * dx
        Y = (J.astype(T) + offs[B]) * dx
        Z = (K.astype(T) + offs[Cc]) * dx
        X, Y, Z = X.ravel(), Y.ravel(), Z.ravel()
    elif ppc == 16:
        rng = _MT19937_64(seed)
        pts = []
        for i in range(i0, i1 + 1):
            for j in range(j0, j1 + 1):
                for k in range(k0, k1 + 1):
                    for _ in range(16):
                        if precision == 4:
                            u, v, w = rng.uniform_f32(), rng.uniform_f32(), rng.uniform_f32()
                        else:
                            u, v, w = rng.uniform(), rng.uniform(), rng.uniform()
                        pts.append(((T(i) + T(u)) * dx, (T(j) + T(v)) * dx, (T(k) + T(w)) * dx))
        arr = np.array(pts, dtype=T).reshape(-1, 3)
        X, Y, Z = arr[:, 0], arr[:, 1], arr[:, 2]
    else:
        raise ConfigError("sample_shape: particles per cell must be 8, 16 or 27")
    m = _shape_mask(shape, X, Y, Z, T)
    return np.stack([X[m], Y[m], Z[m]], axis=1)


def seed_particles(cfg: SceneConfig, precision: int = 8, i_range: Optional[tuple] = None,
                   allow_empty: bool = False) -> np.ndarray:
    """seed_particles (scene.hpp:204-230) -> Particle<T> structured array.

    i_range: only the lattice x-cells lo..hi of every body (sample_shape),
    i.e. that part of the global emission order (x-slab ranks seed their own
    slab without ever holding the whole set)."""
    T = _T(precision)
    dx = cfg.dx(precision)
    parts = []
    for body in cfg.bodies:
        mat = cfg.materials[body.material]
        xs = sample_shape(body.shape, dx, body.ppc, body.seed, precision, i_range)
        cell_vol = dx * dx * dx
        vol = cell_vol / T(body.ppc)
        mass = T(mat.density) * vol
        p = np.zeros(len(xs), dtype=abi.particle_dtype(precision))
        p["x"] = xs
        v = np.empty_like(xs)
        v[:] = np.array(body.velocity, dtype=T)
        if T(body.shear_slope) != 0:
            v[:, 0] += T(body.shear_slope) * (xs[:, 1] - T(body.shape.center[1]))
        om = np.array(body.omega, dtype=T)
        if T((om[0] * om[0] + om[1] * om[1]) + om[2] * om[2]) > 0:
            c = np.array(body.shape.center, dtype=T)
            r = xs - c
            cr = np.stack([om[1] * r[:, 2] - om[2] * r[:, 1], om[2] * r[:, 0] - om[0] * r[:, 2],
                           om[0] * r[:, 1] - om[1] * r[:, 0]], axis=1)
            v = v + cr
        p["v"] = v
        p["F"] = np.eye(3, dtype=T)
        p["J"] = T(1)
        p["mass"] = mass
        p["volume0"] = vol
        p["material"] = body.material
        parts.append(p)
    out = np.concatenate(parts) if parts else np.zeros(0, dtype=abi.particle_dtype(precision))
    if len(out) == 0 and not allow_empty:
        raise ConfigError("bodies: seeding produced no particles")
    return out


def mass_epsilon(particles: np.ndarray, precision: int = 8) -> float:
    """compute_mass_epsilon: 1e-12 x median mass via nth_element (simulation.hpp:227-232)."""
    T = _T(precision)
    m = np.asarray(particles["mass"])
    if len(m) == 0:
        raise ConfigError("no particles")
    k = len(m) // 2
    return float(T(1e-12) * np.partition(m, k)[k])


def to_abi_config(cfg: SceneConfig, precision: int = 8, mass_eps: float = 0.0,
                  device: int = 0) -> abi.Config:
    """Flatten SimConfig<T> into the C-ABI ckg_config (include/ckmpm_b200.h)."""
    T = _T(precision)
    c = abi.Config()
    c.abi_version = abi.ABI_VERSION
    c.precision = precision
    c.resolution = cfg.resolution
    c.scheme = abi.SCHEME_NAMES[cfg.scheme]
    dx = cfg.dx(precision)
    c.extent = float(T(cfg.extent))
    c.dx = float(dx)
    c.inv_dx = float(T(1) / dx)  # simulation.hpp:250, grid.hpp:117
    for a in range(3):
        c.gravity[a] = float(T(cfg.gravity[a]))
    c.mass_eps = float(mass_eps)
    c.clamp_singular = int(cfg.clamp_singular)
    c.deterministic = int(cfg.deterministic)
    c.clamp_floor = float(T(cfg.clamp_floor))
    if len(cfg.materials) > abi.MAX_MATERIALS:
        raise ConfigError("materials: more than the device table holds")
    c.n_materials = len(cfg.materials)
    for i, m in enumerate(cfg.materials):
        d = c.materials[i]
        d.model = abi.MODEL_NAMES[m.model]
        d.density, d.E, d.nu = float(T(m.density)), float(T(m.E)), float(T(m.nu))
        d.mu, d.lambda_ = float(m.mu), float(m.lam)
        d.bulk, d.gamma, d.viscosity = float(T(m.bulk)), float(T(m.gamma)), float(T(m.viscosity))
        d.friction_angle_deg, d.dp_alpha = float(T(m.friction_angle_deg)), float(m.dp_alpha)
    if len(cfg.boundaries) > abi.MAX_BOUNDARIES:
        raise ConfigError("boundaries: more than the device table holds")
    c.n_boundaries = len(cfg.boundaries)
    for i, b in enumerate(cfg.boundaries):
        d = c.boundaries[i]
        d.kind = abi.BC_NAMES[b.kind]
        for a in range(3):
            d.lo[a], d.hi[a] = float(T(b.lo[a])), float(T(b.hi[a]))
            d.normal[a] = float(T(b.normal[a]))
            d.velocity[a], d.omega[a], d.center[a] = float(T(b.velocity[a])), float(T(b.omega[a])), float(T(b.center[a]))
    c.flags = abi.FLAG_QUADRATIC if cfg.kernel == "quadratic" else 0
    c.device = device
    return c


def block_scene(n_cells: int, resolution: int = 512, scheme: str = "apic",
                model: str = "fixed_corotated", E: float = 1e5, nu: float = 0.4,
                density: float = 1000.0, gravity=(0.0, -9.8, 0.0), y0: float = 0.0625,
                boundary: Optional[str] = "sticky", kernel: str = "compact") -> SceneConfig:
    """SURVEY Appendix C 'C5_block_n' family: FC block of n^3 cells at res 512."""
    h = (n_cells / 2) / resolution
    lo = (0.5 - h, y0, 0.5 - h)
    hi = (lo[0] + n_cells / resolution, y0 + n_cells / resolution, lo[2] + n_cells / resolution)
    mats = [{"model": model, "density": density, "E": E, "nu": nu}]
    if model == "drucker_prager":
        mats[0]["friction_angle_deg"] = 30.0
    obj = {"name": f"C5_block_{n_cells}", "resolution": resolution, "scheme": scheme, "kernel": kernel,
           "gravity": list(gravity), "materials": mats,
           "bodies": [{"shape": {"kind": "box", "lo": list(lo), "hi": list(hi)}, "material": 0, "ppc": 8}],
           "boundaries": []}
    if boundary == "sticky":
        obj["boundaries"] = [{"kind": "sticky", "lo": [0, 0, 0], "hi": [1, y0, 1]}]
    elif boundary == "separate":
        obj["boundaries"] = [{"kind": "separate", "lo": [0, 0, 0], "hi": [1, y0, 1], "normal": [0, 1, 0]}]
    return SceneConfig.from_json(obj)
