"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no kernel, quadrature, tree,
ACA or transform).  It only produces the inputs the paper's experiments are
shaped like (flat-triangle sphere meshes, "approximates the
sphere of radius 1 with M flat triangles"; densities; the plane-wave pulse of
BASELINE.json configs[0]).  The recipes are pinned in SURVEY.md §8(d) and
DESIGN.md "Input recipe":

* icosahedron: cyclic permutations of (0, +-1, +-phi), normalised, 20 outward
  counter-clockwise faces;
* subdivision: (a,b,c) -> (a,ab,ca), (b,bc,ab), (c,ca,bc), (ab,bc,ca), edge
  midpoints projected to the unit sphere and numbered in first-encounter order;
* ellipsoid: vertices scaled after the last subdivision;
* config 5 ("D12"): two unit spheres centred at (+-1.5,0,0), icosphere
  subdivision 6, each face split 1->2 along the median from its first vertex;
* seeds: numpy Generator(PCG64(200605186 + cfg)).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 200605186


def icosahedron():
    """Unit icosahedron: 12 vertices, 20 outward CCW faces."""
    phi = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([
        [-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
        [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
        [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1],
    ], dtype=np.float64)
    v /= np.linalg.norm(v, axis=1)[:, None]
    f = np.array([
        [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
        [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
        [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
        [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
    ], dtype=np.int32)
    return v, f


def _subdivide(v, f):
    verts = [tuple(x) for x in v]
    cache = {}
    out = np.empty((4 * len(f), 3), dtype=np.int32)

    def mid(a, b):
        key = (a, b) if a < b else (b, a)
        idx = cache.get(key)
        if idx is None:
            m = (np.asarray(verts[a]) + np.asarray(verts[b])) * 0.5
            m = m / np.linalg.norm(m)
            idx = len(verts)
            verts.append(tuple(m))
            cache[key] = idx
        return idx

    for t, (a, b, c) in enumerate(f):
        ab = mid(a, b)
        bc = mid(b, c)
        ca = mid(c, a)
        out[4 * t + 0] = (a, ab, ca)
        out[4 * t + 1] = (b, bc, ab)
        out[4 * t + 2] = (c, ca, bc)
        out[4 * t + 3] = (ab, bc, ca)
    return np.asarray(verts, dtype=np.float64), out


def icosphere(subdiv: int):
    """Unit icosphere with 20*4**subdiv flat triangles (vertices on the sphere)."""
    v, f = icosahedron()
    for _ in range(subdiv):
        v, f = _subdivide(v, f)
    return np.ascontiguousarray(v), np.ascontiguousarray(f)


def ellipsoid(subdiv: int, axes=(2.0, 1.0, 0.5)):
    v, f = icosphere(subdiv)
    return np.ascontiguousarray(v * np.asarray(axes, dtype=np.float64)[None, :]), f


def split_median(v, f):
    """Replace each face (a,b,c) by (a,b,m),(a,m,c), m=(b+c)/2 not projected."""
    nv = len(v)
    m = 0.5 * (v[f[:, 1]] + v[f[:, 2]])
    midx = nv + np.arange(len(f), dtype=np.int32)
    out = np.empty((2 * len(f), 3), dtype=np.int32)
    out[0::2, 0] = f[:, 0]
    out[0::2, 1] = f[:, 1]
    out[0::2, 2] = midx
    out[1::2, 0] = f[:, 0]
    out[1::2, 1] = midx
    out[1::2, 2] = f[:, 2]
    return np.ascontiguousarray(np.concatenate([v, m])), out


def two_spheres(subdiv: int = 6, centre: float = 1.5, split: bool = True):
    v, f = icosphere(subdiv)
    if split:
        v, f = split_median(v, f)
    va = v + np.array([-centre, 0.0, 0.0])
    vb = v + np.array([centre, 0.0, 0.0])
    return (np.ascontiguousarray(np.concatenate([va, vb])),
            np.ascontiguousarray(np.concatenate([f, f + len(v)]).astype(np.int32)))


# BASELINE.json configs; T = 2 for every config (reading AM3).
CONFIGS = {
    1: dict(mesh=("icosphere", 2), N=32, T=2.0, leaf=10 ** 9, eta=1.0, m=1, eps=1e-6, dense=True),
    2: dict(mesh=("icosphere", 4), N=128, T=2.0, leaf=32, eta=1.0, m=3, eps=1e-6, dense=False),
    3: dict(mesh=("ellipsoid", 5), N=256, T=2.0, leaf=48, eta=1.0, m=4, eps=1e-7, dense=False),
    4: dict(mesh=("icosphere", 6), N=512, T=2.0, leaf=64, eta=1.0, m=4, eps=1e-6, dense=False),
    5: dict(mesh=("two_spheres", 6), N=1024, T=2.0, leaf=64, eta=1.0, m=5, eps=1e-8, dense=False),
}


def make_mesh(kind: str, level: int):
    if kind == "icosphere":
        return icosphere(level)
    if kind == "ellipsoid":
        return ellipsoid(level)
    if kind == "two_spheres":
        return two_spheres(level)
    raise ValueError(kind)


def config_mesh(cfg: int):
    kind, level = CONFIGS[cfg]["mesh"]
    return make_mesh(kind, level)


def rng(cfg: int, stream: int = 0):
    return np.random.Generator(np.random.PCG64(SEED_BASE + cfg + 1000 * stream))


def random_density(cfg: int, L: int, M: int, stream: int = 0):
    """x_l[i] = a + ib, a,b ~ N(0,1) iid, shape [L][M] complex128 (input panel order)."""
    a = rng(cfg, stream).standard_normal((L, M, 2))
    return np.ascontiguousarray(a[..., 0] + 1j * a[..., 1])


def random_time_data(cfg: int, N: int, M: int, stream: int = 0):
    return np.ascontiguousarray(rng(cfg, stream).standard_normal((N + 1, M)))


def vertex_mean_points(v, f):
    """Arithmetic mean of the three vertices (input-data helper for the pulse)."""
    return (v[f[:, 0]] + v[f[:, 1]] + v[f[:, 2]]) / 3.0


def pulse(v, f, N: int, T: float, shift: float = 1.0, width: float = 0.2):
    """g_n[i] = exp(-((t_n - x_i . d - shift)/width)^2), d = (1,0,0), t_n = n T/N.

    BASELINE.json configs[0] plane-wave pulse, evaluated at panel vertex means.
    """
    x = vertex_mean_points(v, f)[:, 0]
    t = np.arange(N + 1, dtype=np.float64) * (T / N)
    return np.ascontiguousarray(np.exp(-(((t[:, None] - x[None, :] - shift) / width) ** 2)))
