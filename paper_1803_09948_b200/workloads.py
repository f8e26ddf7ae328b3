"""Seeded synthetic inputs for the BASELINE.json configs.

The reference measures on no public dataset; every config is a fully specified synthetic point
cloud.  Points and charges are generated once on the host in FP64 and the *same arrays* are fed to
the CPU checker and to the CUDA path.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class FmmConfig:
    """One BASELINE.json matvec configuration.

    ``kd_max`` and ``leaf_cap`` are not named in BASELINE.json but change the interaction lists
    (SURVEY.md §8d); we pin them to what the reference's solver path uses
    (``TraversalConfig::kd_max = 1.0``, traversal.hpp:15; cap ``kd_max/|k|``, solver.cpp:238-242).
    """

    name: str
    n: int
    distribution: str  # "sphere" | "plummer"
    k: float
    order: int
    ncrit: int = 64
    theta: float = 0.4
    kd_max: float = 1.0
    leaf_cap: float = -1.0  # < 0: kd_max/|k| (solver.cpp:238-242); 0: no cap
    seed: int = 12345
    plummer_a: float = 0.05

    def resolved_leaf_cap(self) -> float:
        if self.leaf_cap >= 0:
            return self.leaf_cap
        return self.kd_max / abs(self.k) if self.kd_max > 0 and self.k != 0 else 0.0


CONFIGS = {
    # configs[0]: the reference's own CPU-runnable case
    "cfg1": FmmConfig("cfg1", 16_384, "sphere", 1.0, 10),
    # configs[1]: the configuration the metric is quoted on at N=1
    "cfg2": FmmConfig("cfg2", 1_048_576, "sphere", 4.0, 12),
    # configs[3]: clustered volume
    "cfg4": FmmConfig("cfg4", 4_194_304, "plummer", 8.0, 14, theta=0.35),
    # configs[4]: scaling run (weak: 4,194,304 per GPU)
    "cfg5": FmmConfig("cfg5", 33_554_432, "sphere", 8.0, 12),
    "cfg5_per_gpu": FmmConfig("cfg5_per_gpu", 4_194_304, "sphere", 8.0, 12),
}


def sphere_points(n: int, seed: int) -> np.ndarray:
    """n points uniform on the unit sphere surface: normalised Gaussian triples."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return np.ascontiguousarray(v, dtype=np.float64)


def plummer_points(n: int, seed: int, a: float = 0.05) -> np.ndarray:
    """Plummer-like cluster in the unit cube: r = a / sqrt(u^(-2/3) - 1), isotropic direction,
    centre (1/2,1/2,1/2), samples outside the cube rejected (cfg 4)."""
    rng = np.random.default_rng(seed)
    out = np.empty((0, 3))
    while out.shape[0] < n:
        m = int((n - out.shape[0]) * 1.2) + 16
        u = rng.uniform(1e-12, 1.0, m)
        r = a / np.sqrt(u ** (-2.0 / 3.0) - 1.0 + 1e-300)
        d = rng.standard_normal((m, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        p = 0.5 + d * r[:, None]
        ok = np.all((p >= 0.0) & (p <= 1.0), axis=1)
        out = np.concatenate([out, p[ok]])
    return np.ascontiguousarray(out[:n], dtype=np.float64)


def charges(n: int, seed: int) -> np.ndarray:
    """complex charges, re and im uniform in [-1, 1]"""
    rng = np.random.default_rng(seed + 7919)
    q = rng.uniform(-1.0, 1.0, (n, 2))
    return np.ascontiguousarray(q[:, 0] + 1j * q[:, 1], dtype=np.complex128)


def make_points(cfg: FmmConfig, n: int | None = None) -> np.ndarray:
    n = cfg.n if n is None else n
    if cfg.distribution == "sphere":
        return sphere_points(n, cfg.seed)
    if cfg.distribution == "plummer":
        return plummer_points(n, cfg.seed, cfg.plummer_a)
    raise ValueError(cfg.distribution)


def icosphere_patches(subdivisions: int, radius: float = 1.0) -> np.ndarray:
    """Curved 6-node triangles of a subdivided icosahedron, midside nodes projected to the sphere.

    Returns (20*4^s, 6, 3): 3 corners then 3 midsides (midside k between corners k and (k+1)%3),
    the node order of the reference's CurvilinearPatch (geometry.hpp:13-20).  Missing from the
    reference; needed for BASELINE config 3.
    """
    t = (1.0 + 5.0 ** 0.5) / 2.0
    verts = np.array(
        [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t],
         [0, -1, -t], [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    verts /= np.linalg.norm(verts, axis=1, keepdims=True)
    faces = np.array(
        [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
         [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
         [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]])
    tri = verts[faces]  # (20, 3, 3)
    for _ in range(subdivisions):
        a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
        ab, bc, ca = a + b, b + c, c + a
        ab /= np.linalg.norm(ab, axis=1, keepdims=True)
        bc /= np.linalg.norm(bc, axis=1, keepdims=True)
        ca /= np.linalg.norm(ca, axis=1, keepdims=True)
        tri = np.concatenate([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                              np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)])
    mids = []
    for e in range(3):
        m = tri[:, e] + tri[:, (e + 1) % 3]
        mids.append(m / np.linalg.norm(m, axis=1, keepdims=True))
    patches = np.concatenate([tri, np.stack(mids, 1)], axis=1) * radius
    return np.ascontiguousarray(patches, dtype=np.float64)


def patch_samples(patches: np.ndarray, sample_ref: np.ndarray) -> np.ndarray:
    """Positions of the interpolation nodes (zeta, eta) of every patch, patch-major — the samples of
    the reference's build_system (solver.cpp:283-294) through its quadratic map
    (geometry.cpp:22-45), evaluated in the same operation order (bit-identical)."""
    patches = np.asarray(patches, dtype=np.float64)
    out = np.zeros((patches.shape[0], len(sample_ref), 3))
    for j, (z, e) in enumerate(np.asarray(sample_ref, dtype=np.float64)):
        l1, l2, l3 = 1.0 - z - e, z, e
        n = [l1 * (2 * l1 - 1), l2 * (2 * l2 - 1), l3 * (2 * l3 - 1), 4 * l1 * l2, 4 * l2 * l3, 4 * l3 * l1]
        r = np.zeros((patches.shape[0], 3))
        for k in range(6):
            r += n[k] * patches[:, k, :]
        out[:, j, :] = r
    return out.reshape(-1, 3)


def mie_soft_sphere(radius: float, k: float, r, theta) -> np.ndarray:
    """Scattered field of the plane wave e^{ikz} off a sound-soft sphere, the classical series
        u_s(r, theta) = - sum_n i^n (2n + 1) j_n(ka) / h_n(ka) h_n(kr) P_n(cos theta)
    (the analytic oracle of BASELINE config 3; the reference carries the same series in
    oracle.cpp:11-59).  r, theta: observation radii (>= radius) and polar angles."""
    from scipy.special import eval_legendre, spherical_jn, spherical_yn

    r, theta = np.broadcast_arrays(np.asarray(r, dtype=np.float64), np.asarray(theta, dtype=np.float64))
    ka = k * radius
    nmax = int(ka + 8.0 * np.cbrt(ka) + 16.0)
    n = np.arange(nmax + 1)
    h = lambda z: spherical_jn(n, z) + 1j * spherical_yn(n, z)
    ratio = spherical_jn(n, ka) / h(ka)
    out = np.zeros(r.shape, dtype=np.complex128)
    for idx in np.ndindex(r.shape):
        out[idx] = -np.sum((2 * n + 1) * (1j ** n) * ratio * h(k * r[idx]) * eval_legendre(n, np.cos(theta[idx])))
    return out



def quadrature_tables(basis_order: int = 1) -> dict:
    """The interpolation / quadrature tables of hfmm_correction_rules for basis order 1 or 2 (near rule 25,
    Duffy rule 8 — the reference's KernelConfig defaults, kernel.hpp:48-50), shipped with the package
    (data/quadrature_rules.npz, tabulated from the reference's geometry.cpp by
    scripts/make_quadrature_tables.py)."""
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "quadrature_rules.npz")
    g = np.load(path)
    prefix = f"order{int(basis_order)}_"
    keys = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")
    if prefix + keys[0] not in g.files:
        raise ValueError("tables are shipped for basis orders 1 and 2")
    return {k: g[prefix + k] for k in keys}
