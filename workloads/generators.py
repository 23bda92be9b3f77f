"""Seeded generators for the BASELINE.json workloads (C1..C5) and test inputs.

Recipe (SURVEY.md §8(d) "Synthetic inputs", readings R1, R22):
  * numpy ``default_rng(seed)``, draws made in the order written in each function;
  * positions computed in fp64, wrapped into [0, L), then quantised to the grid
    L * 2**-24 and stored as fp32 (exact), so periodic shifts by whole grid
    steps are exact in fp32;
  * v, u, m, h0 stored as fp32 (round to nearest);
  * arrays: x[N,3] v[N,3] m[N] u[N] h0[N] (h0 == 0 means "library guess").

Seeds 140423031..140423035 are C1..C5, 140423036 SC-exact, 140423037 FCC-exact,
140423100+t the tiny configs.

No SPH arithmetic lives here (no kernel, no neighbour search): the h0 values
are the configs' stated initial guesses, not solutions.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

GRID_BITS = 24


@dataclasses.dataclass
class Particles:
    name: str
    box: tuple            # (Lx, Ly, Lz)
    x: np.ndarray         # [N,3] fp32
    v: np.ndarray         # [N,3] fp32
    m: np.ndarray         # [N]   fp32
    u: np.ndarray         # [N]   fp32
    h0: np.ndarray        # [N]   fp32 (0 = library guess)
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    def take(self, idx) -> "Particles":
        idx = np.asarray(idx)
        return Particles(self.name, self.box, self.x[idx].copy(), self.v[idx].copy(),
                         self.m[idx].copy(), self.u[idx].copy(), self.h0[idx].copy(),
                         dict(self.meta))


def quantise_positions(x64: np.ndarray, box) -> np.ndarray:
    """Wrap fp64 positions into [0,L) and snap them to the L*2^-24 grid (exact in fp32)."""
    box = np.asarray(box, dtype=np.float64)
    x = np.mod(x64, box)
    k = np.floor(x / box * (1 << GRID_BITS))
    k = np.where(k >= (1 << GRID_BITS), 0.0, k)          # x == L after rounding -> 0
    k = np.where(k < 0, 0.0, k)
    xq = (k * (box / (1 << GRID_BITS))).astype(np.float32)
    assert np.all(xq.astype(np.float64) == k * (box / (1 << GRID_BITS)))
    return xq


def _pack(name, box, x64, v, m, u, h0, **meta) -> Particles:
    n = x64.shape[0]
    return Particles(name, tuple(float(b) for b in box), quantise_positions(x64, box),
                     np.ascontiguousarray(v, dtype=np.float32).reshape(n, 3),
                     np.ascontiguousarray(np.broadcast_to(m, (n,)), dtype=np.float32),
                     np.ascontiguousarray(np.broadcast_to(u, (n,)), dtype=np.float32),
                     np.ascontiguousarray(np.broadcast_to(h0, (n,)), dtype=np.float32),
                     meta)


# ---------------------------------------------------------------- C1 ------------
def c1(seed: int = 140423031, n: int = 32768) -> Particles:
    """BASELINE configs[0]: uniform random in the periodic unit box.

    v ~ N(0, 0.01) per component (std, R22), u = 1, m = 1/N,
    h0 = 1.2348 * 1.825742 * N^(-1/3) (R1: 1.2348 is an eta with support
    1.825742*h; the paper's h is the support radius).
    """
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    v = rng.normal(0.0, 0.01, (n, 3))
    h0 = 1.2348 * 1.825742 * n ** (-1.0 / 3.0)
    return _pack("C1", (1.0, 1.0, 1.0), x, v, 1.0 / n, 1.0, h0, seed=seed)


# ---------------------------------------------------------------- lattices ------
def _sc_lattice(k: int) -> np.ndarray:
    i = np.arange(k, dtype=np.float64)
    g = np.stack(np.meshgrid(i, i, i, indexing="ij"), axis=-1).reshape(-1, 3)
    return (g + 0.5) / k


def c2(seed: int = 140423032, k: int = 64, jitter: float = 0.1) -> Particles:
    """BASELINE configs[1]: k^3 cubic lattice jittered by U(-0.1,0.1)*spacing."""
    rng = np.random.default_rng(seed)
    x = _sc_lattice(k)
    n = x.shape[0]
    if jitter:
        x = x + rng.uniform(-jitter, jitter, (n, 3)) / k
    h0 = 2.2515 / k
    return _pack("C2" if jitter else "C2-exact", (1.0, 1.0, 1.0), x, np.zeros((n, 3)),
                 1.0 / n, 1.0, h0, seed=seed, spacing=1.0 / k)


def c2_exact(k: int = 64) -> Particles:
    """Perfect SC lattice (closed-form parity case)."""
    p = c2(seed=140423036, k=k, jitter=0.0)
    p.name = "SC-exact"
    return p


def fcc_exact(k: int = 32) -> Particles:
    """Perfect FCC lattice, k^3 cubes x 4 sites (Sedov lattice type)."""
    base = _sc_lattice(k) - 0.5 / k                    # cube corners i/k
    offs = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]]) / k
    x = (base[:, None, :] + offs[None, :, :]).reshape(-1, 3) + 0.25 / k
    n = x.shape[0]
    dbar = n ** (-1.0 / 3.0)
    return _pack("FCC-exact", (1.0, 1.0, 1.0), x, np.zeros((n, 3)), 1.0 / n, 1.0,
                 2.2587 * dbar, seed=140423037, spacing=dbar)


# ---------------------------------------------------------------- C3 ------------
def c3(seed: int = 140423033, kl: int = 96, kr: int = 48, jitter: float = 0.1) -> Particles:
    """BASELINE configs[2] (Sod-like, R22): box 2x1x1, left kl^3 lattice in [0,1)^3,
    right kr^3 lattice in [1,2)x[0,1)^2, jitter U(-0.1,0.1)*local spacing,
    m = 1.125/N (rho_L = 1, rho_R = 0.125 for kl = 2*kr), u = 2.5 | 2.0, v = 0."""
    rng = np.random.default_rng(seed)
    xl = _sc_lattice(kl)
    xr = _sc_lattice(kr)
    xr[:, 0] += 1.0
    xl = xl + rng.uniform(-jitter, jitter, xl.shape) / kl
    xr = xr + rng.uniform(-jitter, jitter, xr.shape) / kr
    x = np.concatenate([xl, xr])
    n = x.shape[0]
    u = np.concatenate([np.full(len(xl), 2.5), np.full(len(xr), 2.0)])
    h0 = np.concatenate([np.full(len(xl), 2.2515 / kl), np.full(len(xr), 2.2515 / kr)])
    m = 1.0 / kl ** 3          # = 1.125/N for kl = 2*kr: rho_L = 1, rho_R = (kr/kl)^3
    return _pack("C3", (2.0, 1.0, 1.0), x, np.zeros((n, 3)), m, u, h0, seed=seed)


# ---------------------------------------------------------------- C4/C5 ---------
def _clustered(name: str, seed: int, n: int, n_clumps: int, box=(1.0, 1.0, 1.0)) -> Particles:
    """Clustered multi-resolution periodic unit box (SURVEY §8(d) C4 recipe):
    (1) floor(0.3N) uniform background; (2) centres U[0,1)^3; (3) scale radii
    a = exp(U(ln 0.002, ln 0.02)); (4) remaining particles split evenly, the
    first (rem) clumps get +1; (5) Plummer radii truncated at 20a:
    X = U*(400/401)^(3/2), r = a / sqrt(X^(-2/3) - 1), isotropic direction
    (z = U(-1,1), phi = U(0, 2pi)); (6) wrap; (7) v ~ N(0, 0.1);
    (8) u = exp(U(ln 0.1, ln 10)); (9) m = 1/N; h0 = 0 (library guess)."""
    rng = np.random.default_rng(seed)
    boxa = np.asarray(box, dtype=np.float64)
    nb = int(math.floor(0.3 * n))
    xb = rng.random((nb, 3)) * boxa
    centres = rng.random((n_clumps, 3)) * boxa
    a = np.exp(rng.uniform(math.log(0.002), math.log(0.02), n_clumps))
    nc = n - nb
    per, rem = divmod(nc, n_clumps)
    counts = np.full(n_clumps, per, dtype=np.int64)
    counts[:rem] += 1
    owner = np.repeat(np.arange(n_clumps), counts)
    X = rng.random(nc) * (400.0 / 401.0) ** 1.5
    r = a[owner] / np.sqrt(X ** (-2.0 / 3.0) - 1.0)
    z = rng.uniform(-1.0, 1.0, nc)
    phi = rng.uniform(0.0, 2.0 * math.pi, nc)
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    xc = centres[owner] + r[:, None] * np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    x = np.concatenate([xb, xc])
    v = rng.normal(0.0, 0.1, (n, 3))
    u = np.exp(rng.uniform(math.log(0.1), math.log(10.0), n))
    return _pack(name, box, x, v, float(np.prod(boxa)) / n, u, 0.0, seed=seed,
                 n_clumps=n_clumps, scale_radii=a.tolist())


def c4(seed: int = 140423034, n: int = 2097152, n_clumps: int = 64) -> Particles:
    """BASELINE configs[3]: 2,097,152 particles, 30% background + 64 Plummer clumps."""
    return _clustered("C4", seed, n, n_clumps)


def c4_weak(replicas: int, seed: int = 140423038) -> Particles:
    """Weak-scaling version of C4 for `replicas` GPUs: box (replicas, 1, 1) with
    replicas x 2,097,152 particles and replicas x 64 clumps (same density, same clump
    statistics); slab decomposition along x gives each GPU about one C4."""
    return _clustered(f"C4x{replicas}", seed, replicas * 2097152, replicas * 64, box=(float(replicas), 1.0, 1.0))


def c5(seed: int = 140423035, n: int = 512 ** 3, n_clumps: int = 512) -> Particles:
    """BASELINE configs[4]: 512^3 particles, same generator with 512 clumps."""
    return _clustered("C5", seed, n, n_clumps)


# ---------------------------------------------------------------- tiny ----------
def tiny(t: int, n: int = 600, clump_frac: float = 0.4, n_dup: int = 3,
         equal_mass: bool = False) -> Particles:
    """Small adversarial mixes for brute-force parity (SURVEY §8(d) 'tiny'):
    a uniform part plus one Gaussian clump centred on the periodic corner
    (so it straddles all three wrap boundaries), h spanning ~100x
    (clump h in [0.002,0.02], background h in [0.08,0.2], log-uniform),
    unequal masses (catches m_i/m_j swaps) and a few exact duplicates
    (coincident pairs, r = 0)."""
    rng = np.random.default_rng(140423100 + t)
    nc = int(round(clump_frac * n))
    nu = n - nc - n_dup
    xu = rng.random((nu, 3))
    xc = rng.normal(0.0, 0.02, (nc, 3))
    x = np.concatenate([xu, xc])
    dup = rng.integers(0, x.shape[0], n_dup)
    x = np.concatenate([x, x[dup]])
    hu = np.exp(rng.uniform(math.log(0.08), math.log(0.2), nu))
    hc = np.exp(rng.uniform(math.log(0.002), math.log(0.02), nc))
    h = np.concatenate([hu, hc])
    h = np.concatenate([h, h[dup]])
    v = rng.normal(0.0, 0.3, (n, 3))
    u = np.exp(rng.uniform(math.log(0.5), math.log(2.0), n))
    m = np.full(n, 1.0 / n) if equal_mass else rng.uniform(0.5, 1.5, n) / n
    return _pack(f"tiny{t}", (1.0, 1.0, 1.0), x, v, m, u, h, seed=140423100 + t)


def edges_unquantised(t: int = 0, n: int = 4000) -> Particles:
    """Arbitrary fp32 positions (NOT snapped to the 2^-24 grid) crowded against the periodic
    faces: 40% of the particles within 2e-3 of x, y or z = 0 or L, including the exact values
    0 and the largest fp32 below L, the rest uniform; unequal masses, random v and u. The
    minimum-image differences across the wrap are then inexact in fp32 (H2): the GPU must
    still match the fp64 oracle within the tolerances."""
    rng = np.random.default_rng(140423200 + t)
    x = rng.random((n, 3))
    k = int(0.4 * n)
    idx = rng.choice(n, k, replace=False)
    ax = rng.integers(0, 3, k)
    side = rng.integers(0, 2, k)
    d = rng.random(k) * 2e-3
    x[idx, ax] = np.where(side == 0, d, 1.0 - d)
    xf = x.astype(np.float32)
    top = np.nextafter(np.float32(1.0), np.float32(0.0))
    xf[idx[:8], ax[:8]] = np.where(side[:8] == 0, np.float32(0.0), top)
    xf = np.where(xf >= np.float32(1.0), top, xf).astype(np.float32)
    v = rng.normal(0.0, 0.2, (n, 3))
    u = np.exp(rng.uniform(math.log(0.5), math.log(2.0), n))
    m = rng.uniform(0.5, 1.5, n) / n
    return Particles(f"edges{t}", (1.0, 1.0, 1.0), np.ascontiguousarray(xf),
                     v.astype(np.float32), m.astype(np.float32), u.astype(np.float32),
                     np.zeros(n, dtype=np.float32), {"seed": 140423200 + t})


CONFIGS = {
    "C1": c1, "C2": c2, "C2-exact": c2_exact, "SC-exact": c2_exact,
    "FCC-exact": fcc_exact, "C3": c3, "C4": c4, "C5": c5,
}


def make(name: str, **kw) -> Particles:
    if name.startswith("tiny"):
        return tiny(int(name[4:] or 0), **kw)
    return CONFIGS[name](**kw)


def subsample_box(p: Particles, frac: float, seed: int = 0) -> np.ndarray:
    """Seeded sample of particle indices (used to pick parity targets)."""
    rng = np.random.default_rng(seed)
    k = max(1, int(round(frac * p.n)))
    return np.sort(rng.choice(p.n, size=k, replace=False))
