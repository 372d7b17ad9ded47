"""Pins of the oracle's time-domain path with compressed weights (SURVEY §8(f)
NEXT-2): eq:fastdft, eq:fastrhs and the
marching-on-in-time recursion eq:cqmrhs with one LU of V^_0
(P:686-703), on the combined skeleton (every block MACA-compressed).

What fixes them without the GPU path:
  * the fast convolution (per block and term: history sum first, then the
    pivot slice) equals the convolution with the densely assembled weights;
  * the exact identity of the R-scaled transforms: forward -> V(s_l) ->
    inverse equals the causal convolution with the same weights plus the
    R^L-damped wrap-around, sum_{k>n} R^L V^_{L+n-k} q_k (the wrap is 1e-6 of
    the result here, the identity holds to 1e-10);
  * the compressed weights converge to the dense-definition weights
    (DFT of the dense collocation matrices, as in test_oracle_pins) with the
    interpolation order m;
  * the MoT solution satisfies the recursion through the fast convolution,
    and agrees with the frequency-decoupled solve up to the O(R^L) wrap.
"""
import numpy as np
import pytest

import oracle as O
import synth

N, TT = 16, 2.0


@pytest.fixture(scope="module")
def setup():
    V, T = synth.icosphere(2)
    R = O.default_R(N)
    s = O.frequencies(N, TT)
    h = O.H2(V, T, 16, 1.0, 3)
    h.aca(s, 1e-8)
    h.aca_near(s, 1e-8)
    h.time_weights(R)
    W = [h.weight_dense(n) for n in range(N + 1)]
    return V, T, R, s, h, W


def test_fast_conv_equals_dense_weights(setup):
    V, T, R, s, h, W = setup
    M, L = len(T), N + 1
    q = np.random.default_rng(1).standard_normal((L, M))
    y = h.conv(q)
    yd = np.array([sum(W[n - k] @ q[k] for k in range(n + 1)) for n in range(L)])
    assert np.linalg.norm(y - yd) / np.linalg.norm(yd) <= 1e-11
    y3 = h.conv(q, kmax=3)
    yd3 = np.array([sum(W[n - k] @ q[k] for k in range(min(n, 3) + 1)) for n in range(L)])
    assert np.linalg.norm(y3 - yd3) / np.linalg.norm(yd3) <= 1e-11


def test_transform_identity_with_wrap(setup):
    V, T, R, s, h, W = setup
    M, L = len(T), N + 1
    q = np.random.default_rng(2).standard_normal((L, M))
    yt = O.inverse(h.apply(O.MODE_COMBINED, s, O.forward(q.astype(complex), N, R)), N, R)
    conv = h.conv(q)
    wrap = np.array([sum((W[L + n - k] @ q[k] for k in range(n + 1, L)), np.zeros(M, complex)) for n in range(L)])
    assert np.linalg.norm(R ** L * wrap) / np.linalg.norm(yt) > 1e-8   # the wrap is visible ...
    assert np.linalg.norm(yt - (conv + R ** L * wrap)) / np.linalg.norm(yt) <= 1e-10   # ... and exactly accounted


def test_compressed_weights_converge_to_dense():
    V, T = synth.icosphere(2)
    L, R = N + 1, O.default_R(N)
    s = O.frequencies(N, TT)
    As = [O.dense_matrix(V, T, sl) for sl in s]
    Vhat = [sum(As[l] * np.exp(2j * np.pi * ((k * l) % L) / L) for l in range(L)) * R ** (-k) / L for k in range(L)]
    e = []
    for m in (2, 3, 4):
        h = O.H2(V, T, 16, 1.0, m)
        h.aca(s, 1e-10)
        h.aca_near(s, 1e-10)
        h.time_weights(R)
        e.append(max(np.linalg.norm(h.weight_dense(n).real - Vhat[n].real) for n in range(L))
                 / np.linalg.norm(Vhat[0].real))
    assert e[0] > 3 * e[1] > 9 * e[2] and e[2] <= 2e-4, e


def test_mot_recursion_and_frequency_solve(setup):
    V, T, R, s, h, W = setup
    g = synth.pulse(V, T, N, TT, shift=2.2)
    q = h.mot(g)
    # the recursion, checked through the other code path (fast convolution)
    res = h.conv(q).real - g
    assert np.linalg.norm(res) <= 1e-11 * np.linalg.norm(g)
    # frequency-decoupled solve of the same compressed operator: equal up to the O(R^L) wrap
    phif, it, rr = h.gmres(O.MODE_COMBINED, s, O.forward(g.astype(complex), N, R), tol=1e-12)
    phi = O.inverse(phif, N, R).real
    assert np.linalg.norm(q - phi) / np.linalg.norm(phi) <= 1e-4
