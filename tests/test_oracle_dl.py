"""Pins of the oracle's double-layer operator K(s) (
eq:wavebio P:301-303: gamma_{1,y} of the fundamental solution P:479-482).

Closed forms used (derived from the kernel, not re-typed from the oracle):
  * unit sphere, constant density, chord measure dS = 2 pi r dr and
    (y - x).n_y = r^2/2:  K(s) 1 = -(1/4) int_0^2 (1 + s r) e^{-s r} dr
                                 = e^{-2s}/2 - (1 - e^{-2s})/(2s)   (-1/2 at s = 0);
  * Gauss's law at s = 0 on any closed surface: K(0) 1 = -1/2;
  * exterior Calderon identity of eq:wavebie for the outgoing
    radial solution e^{-s|x|}/|x| on the unit sphere: V(s) q = (-1/2 + K(s)) g
    with g = e^{-s}, q = -(1 + s) e^{-s}.
"""
import numpy as np
import pytest
from scipy.integrate import dblquad

import oracle as O
import synth


def kappa0(s):
    s = complex(s)
    if s == 0:
        return -0.5
    return 0.5 * np.exp(-2 * s) - (1 - np.exp(-2 * s)) / (2 * s)


def lambda0(s):
    s = complex(s)
    return 1.0 if s == 0 else (1 - np.exp(-2 * s)) / (2 * s)


@pytest.mark.parametrize("s", [0.0, 1.3, 5.57, 2 + 3j])
def test_dl_sphere_eigenvalue_converges(s):
    errs = []
    for sub in (2, 3, 4):
        V, T = synth.icosphere(sub)
        h = O.H2(V, T, 10 ** 6, 1.0, 1)
        y = h.apply_dl(O.MODE_DENSE, np.array([s]), np.ones((1, len(T)), complex), np.array([0], np.int32))[0]
        errs.append(np.max(np.abs(y - kappa0(s))) / abs(kappa0(s)))
    order = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert min(order) >= 0.8, (errs, order)
    assert errs[-1] <= 6e-3, errs


def test_dl_gauss_law_ellipsoid():
    V, T = synth.ellipsoid(3)
    y = O.dense_matrix_dl(V, T, 0.0) @ np.ones(len(T))
    assert np.mean(np.abs(y + 0.5)) <= 5e-3 and np.max(np.abs(y + 0.5)) <= 3e-2


def test_dl_calderon_exterior_sphere():
    """V q = (-1/2 + K) g for the outgoing radial solution (both operators discrete)."""
    V, T = synth.icosphere(4)
    M = len(T)
    h = O.H2(V, T, 10 ** 6, 1.0, 1)
    for s in (1.0, 4.0, 3 + 2j):
        g = np.full((1, M), np.exp(-s), complex)
        q = -(1 + s) * g
        lhs = h.apply(O.MODE_DENSE, np.array([s]), q, np.array([0], np.int32))[0]
        rhs = h.apply_dl(O.MODE_DENSE, np.array([s]), g, np.array([0], np.int32), alpha=-0.5)[0]
        assert np.max(np.abs(lhs - rhs)) / np.max(np.abs(rhs)) <= 1e-2, s


def test_dl_entries_structure():
    V, T = synth.icosphere(2)
    K = O.dense_matrix_dl(V, T, 3.0)
    assert np.all(np.diag(K) == 0)
    assert np.all(K.imag == 0)                     # real s -> real matrix
    K1 = O.dense_matrix_dl(V, T, 2 + 5j)
    K2 = O.dense_matrix_dl(V, T, 2 - 5j)
    assert np.array_equal(K2, np.conj(K1))         # K(conj s) = conj K(s)
    n = O.normals(V, T)
    assert np.allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-14)
    cen = synth.vertex_mean_points(V, T)
    assert np.all(np.sum(n * cen, axis=1) > 0)     # icosphere faces are outward CCW


def test_dl_regular_entry_vs_adaptive_quadrature():
    """One regular entry against scipy's adaptive 2-D quadrature of the kernel
    over the source triangle; error falls like (diam/dist)^5 or faster."""
    A, B, Cv = np.array([0.0, 0, 0]), np.array([0.2, 0, 0]), np.array([0.05, 0.17, 0])
    n = np.array([0.0, 0.0, 1.0])
    s = 2.0 + 1.0j
    errs = []
    for dist in (0.6, 1.2, 2.4):
        x = np.array([0.08, 0.05, 0.0]) + dist * np.array([0.3, 0.2, 0.9]) / np.linalg.norm([0.3, 0.2, 0.9])
        V = np.array([A, B, Cv, x + np.array([0, 0, 0.01]), x + np.array([0.01, 0, 0]), x + np.array([0, 0.01, 0])])
        T = np.array([[3, 4, 5], [0, 1, 2]], dtype=np.int32)
        c0 = (V[3] + V[4] + V[5]) / 3.0
        K = O.dense_matrix_dl(V, T, s)

        def f(v, u, part):
            y = A + u * (B - A) + v * (Cv - A)
            d = y - c0
            r = np.linalg.norm(d)
            val = -(1 + s * r) * np.exp(-s * r) * np.dot(d, n) / (4 * np.pi * r ** 3)
            return (val.real if part == 0 else val.imag)
        jac = np.linalg.norm(np.cross(B - A, Cv - A))
        ref = sum((1j if part else 1.0) * dblquad(f, 0, 1, 0, lambda u: 1 - u, args=(part,), epsabs=1e-13,
                                                   epsrel=1e-12)[0] for part in (0, 1)) * jac
        errs.append(abs(K[0, 1] - ref) / abs(ref))
    assert errs[-1] < errs[0] and errs[0] < 1e-5, errs
    assert np.log2(errs[0] / errs[2]) / 2 >= 4.0, errs


def test_dl_h2_error_decays_with_m_and_aca_limit():
    V, T = synth.icosphere(3)
    s = O.frequencies(32, 2.0)
    x = synth.random_density(2, 3, len(T))
    lsel = np.array([0, 5, 16], np.int32)
    e = []
    for m in (2, 3, 4):
        h = O.H2(V, T, 32, 1.0, m)
        yd = h.apply_dl(O.MODE_DENSE, s, x, lsel)
        yo = h.apply_dl(O.MODE_H2ONLY, s, x, lsel)
        e.append(np.linalg.norm(yo - yd) / np.linalg.norm(yd))
    assert e[0] > 3 * e[1] > 9 * e[2], e
    h = O.H2(V, T, 32, 1.0, 3)
    h.aca(s, 1e-12)
    ya = h.apply_dl(O.MODE_H2ACA, s, x, lsel)
    yo = h.apply_dl(O.MODE_H2ONLY, s, x, lsel)
    assert np.linalg.norm(ya - yo) / np.linalg.norm(yo) <= 1e-11
