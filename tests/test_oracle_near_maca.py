"""Pins of the oracle's near-field MACA (Alg. 3 NEAR branch, P:1426-1431 and
P:1444-1450; eq:lrfinal P:1404-1410 for b in P-).

What fixes it without the GPU path:
  * the pinned entries it reads equal the C3 definition (libm tier, itself
    pinned by test_oracle_pins) to a few ulps, self panels included;
  * the pinned expm1 against math.expm1;
  * the reading k_1 = 0 makes l = 0 a pivot frequency of every block and the
    residual fibre vanishes exactly there, so at l = 0 the combined apply IS
    the exact near field (a transposed Z, a wrong slice or a wrong block
    offset breaks this);
  * L = 1: every near block has rank 1 and the skeleton is the block itself;
  * the combined apply converges to the H2ACA apply (near field exact) as
    eps -> 0, with error below eps (Corollary P:1461-1470 for the near part).
"""
import math

import numpy as np

import oracle as O
import synth


def test_pinned_entries_match_definition():
    V, T = synth.icosphere(2)
    for s in (0.0, 1.0, 3 + 2j, 40 - 25j, 240 + 127j):
        A = O.dense_matrix(V, T, s)
        B = O.dense_matrix_pinned(V, T, s)
        rel = np.abs(A - B) / np.abs(A)
        assert rel.max() <= 2e-15, (s, rel.max())
        d = np.abs(np.diag(A) - np.diag(B)) / np.abs(np.diag(A))
        assert d.max() <= 2e-15, (s, d.max())
    # real s -> real pinned matrix, conj symmetry of the definition
    assert np.all(O.dense_matrix_pinned(V, T, 2.5).imag == 0.0)


def test_pinned_expm1():
    xs = np.concatenate([-np.logspace(-12, np.log10(0.49), 60), [-0.5, -0.7, -1.0, -3.0, -30.0],
                         np.logspace(-12, np.log10(0.49), 20)])
    for x in xs:
        ref = math.expm1(x)
        assert abs(O.pexpm1(x) - ref) <= 4e-16 * abs(ref), x


def _setup(L_N=16, sub=3, nmin=32, m=3):
    V, T = synth.icosphere(sub)
    s = O.frequencies(L_N, 2.0)
    h = O.H2(V, T, nmin, 1.0, m)
    return V, T, s, h


def test_combined_equals_exact_near_at_l0():
    V, T, s, h = _setup()
    L = len(s)
    h.aca(s, 1e-8)
    r = h.aca_near(s, 1e-3)                       # deliberately coarse: l = 0 must still be exact
    assert np.all(r["pivots"][np.r_[0, np.cumsum(r["ranks"])[:-1]], 0] == 0)   # k_1 = 0 in every block
    x = synth.random_density(2, 1, len(T))
    ya = h.apply(O.MODE_H2ACA, s, x, np.array([0], np.int32))
    yc = h.apply(O.MODE_COMBINED, s, x, np.array([0], np.int32))
    assert np.linalg.norm(yc - ya) / np.linalg.norm(ya) <= 1e-14
    # at another frequency the coarse skeleton is visibly approximate
    x5 = synth.random_density(2, 1, len(T), stream=1)
    l5 = np.array([5], np.int32)
    e5 = np.linalg.norm(h.apply(O.MODE_COMBINED, s, x5, l5) - h.apply(O.MODE_H2ACA, s, x5, l5))
    assert e5 / np.linalg.norm(h.apply(O.MODE_H2ACA, s, x5, l5)) > 1e-8


def test_single_frequency_rank_one():
    V, T = synth.icosphere(2)
    s = np.array([4.0 + 0j])
    h = O.H2(V, T, 16, 1.0, 2)
    h.aca(s, 1e-6)
    r = h.aca_near(s, 1e-6)
    assert np.all(r["ranks"] == 1) and np.all(r["Z"] == 1.0)
    x = synth.random_density(2, 1, len(T))
    ya = h.apply(O.MODE_H2ACA, s, x)
    yc = h.apply(O.MODE_COMBINED, s, x)
    assert np.linalg.norm(yc - ya) / np.linalg.norm(ya) <= 1e-14


def test_combined_converges_with_eps():
    V, T, s, h = _setup()
    L = len(s)
    h.aca(s, 1e-12)
    lsel = np.array([1, 4, 8, 12, 16], np.int32)
    x = synth.random_density(2, len(lsel), len(T))
    ya = h.apply(O.MODE_H2ACA, s, x, lsel)
    errs, ranks = [], []
    for eps in (1e-3, 1e-6, 1e-9, 1e-12):
        r = h.aca_near(s, eps)
        yc = h.apply(O.MODE_COMBINED, s, x, lsel)
        errs.append(np.linalg.norm(yc - ya) / np.linalg.norm(ya))
        ranks.append(r["ranks"].mean())
        assert errs[-1] <= eps, (eps, errs)
        assert r["ranks"].max() <= L
    assert errs[0] > 100 * errs[1] > 1e4 * errs[2], errs
    assert ranks == sorted(ranks), ranks
