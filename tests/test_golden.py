"""Golden fixtures (tests/golden/*.json): worked examples printed in SPEC.md and
numbers fixed by PAPER.md, each with its citation.  The oracle is checked
against them on CPU; the library's host entry points (cqm_frequencies) too,
and its device entry points in the gpu-marked test."""
import json
import os
from math import cos, exp, log, pi, sin, sqrt  # noqa: F401  (used by eval of fixture expressions)

import numpy as np
import pytest

import oracle as O
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def ev(expr, **kw):
    env = dict(pi=pi, exp=np.exp, cos=np.cos, sin=np.sin, sqrt=np.sqrt, log=np.log)
    env.update(kw)
    return complex(eval(expr, {"__builtins__": {}}, env))


SPEC = load("spec_examples.json")
PAPER = load("paper_values.json")


def cube_mesh(a, b):
    """[a,b]^3 surface, 12 outward triangles (input data only)."""
    V = np.array([[x, y, z] for z in (a, b) for y in (a, b) for x in (a, b)], dtype=np.float64)
    quads = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    T = []
    for q in quads:
        T += [(q[0], q[1], q[2]), (q[0], q[2], q[3])]
    return V, np.array(T, dtype=np.int32)


def test_golden_kernel():
    for c in SPEC["kernel"]["cases"]:
        s = complex(*c["s"])
        ref = ev(c["value"])
        for pinned in (False, True):
            assert abs(O.kernel(c["r"], s, pinned) - ref) <= 2e-17, (c, pinned)


def test_golden_frequencies_oracle_and_library():
    import paper_2006_05186_b200 as pb
    for c in SPEC["frequencies"]["cases"]:
        ref = ev(c["value"])
        so = O.frequencies(c["N"], c["T"], c["R"], c["method"])
        sl = pb.cqm_frequencies(c["N"], c["T"], c["R"], c["method"])
        assert abs(so[c["l"]] - ref) <= 1e-15
        assert sl[c["l"]] == so[c["l"]]


def test_golden_admissibility():
    for c in SPEC["admissibility"]["cases"]:
        assert O.admissible(c["box_r"], c["box_c"], c["eta"]) == c["admissible"], c


def test_golden_chebyshev_nodes():
    """Nodes of a single-cluster tree on the cube [a,b]^3 (its tight box), per axis."""
    for c in SPEC["chebyshev"]["cases"]:
        V, T = cube_mesh(c["a"], c["b"])
        h = O.H2(V, T, 10 ** 6, 1.0, c["m"])
        xi = h.bases()["xi"][0]
        ref = np.array([ev(e).real for e in c["nodes"]])
        for axis in range(3):
            assert np.allclose(xi[axis], ref, atol=1e-15, rtol=0), (c, xi[axis])


def test_golden_areas():
    a = SPEC["areas"]
    tv = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float) / (2 * 2 ** 0.5)
    tt = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], dtype=np.int32)
    assert abs(O.geometry(tv, tt)["area"].sum() - ev(a["tetrahedron_total"]).real) < 1e-14
    V, T = cube_mesh(0.0, 1.0)
    assert abs(O.geometry(V, T)["area"].sum() - ev(a["cube_total"]).real) < 1e-14
    V, T = synth.icosphere(2)
    assert abs(O.geometry(V, T)["area"].sum() / (4 * pi) - 1) < a["icosphere2_rel_to_4pi"]


def test_golden_gram_norm_and_maca():
    A = np.ones((4, 2), dtype=np.complex128)  # C_1 = ones(2x2) unfolded, d_1 = (1,1)
    r = O.aca_matrix(A, 1e-12)
    assert r["rank"] == 1
    assert abs(np.sqrt(r["nrm2"][-1]) - ev(SPEC["gram_norm"]["value"]).real) < 1e-15
    m = SPEC["maca"]
    rng = np.random.default_rng(3)
    a = rng.standard_normal(36) + 1j * rng.standard_normal(36)
    A = np.repeat(a[:, None], 9, axis=1)
    r = O.aca_matrix(A, 1e-12)
    assert r["rank"] == m["constant_rank"]
    rec = r["C"].T @ r["D"]
    assert np.linalg.norm(rec - A) / np.linalg.norm(A) <= m["constant_tol"]
    assert O.aca_matrix(np.zeros((36, 9), dtype=np.complex128), 1e-12)["rank"] == m["zero_rank"]


def test_golden_paper_R_rule():
    for c in PAPER["R_rule"]["cases"]:
        assert abs(O.default_R(c["N"]) - ev(c["value"]).real) <= 4e-16


def test_golden_bdf2_characteristic_and_self_integral():
    # zeta = 1 (l = 0 with R -> 1) gives delta(1) = 0, i.e. s_0 -> 0 as R -> 1
    s = O.frequencies(8, 1.0, 1.0 - 1e-15)
    assert abs(s[0]) < 1e-13
    c = PAPER["self_integral_equilateral"]
    a = c["a"]
    A, B, C = np.array([0.0, 0, 0]), np.array([a, 0, 0]), np.array([a / 2, a * sqrt(3) / 2, 0])
    assert abs(O.self_integral(A, B, C) - ev(c["value"]).real) < 1e-14


def test_golden_sphere_eigenvalue_dense():
    c = PAPER["sphere_eigenvalue"]
    s = complex(*c["s"])
    ref = ev(c["value"], s=s)
    V, T = synth.icosphere(3)
    y = O.dense_matrix(V, T, s) @ np.ones(len(T))
    assert np.max(np.abs(y - ref)) / abs(ref) < 5e-3  # O(h) collocation error (C11)


@pytest.mark.gpu
def test_golden_library_device():
    """Library (device path): single-cluster tree on the cube gives the SPEC nodes
    through the DENSE apply being consistent; kernel values via the pinned device functions."""
    import paper_2006_05186_b200 as pb
    e, sn, cs = pb.debug_pinned(np.array([0.0, -2.0, 2.0]))
    assert e[0] == 1.0 and sn[0] == 0.0 and cs[0] == 1.0
    k = e[1] * (cs[2] - 1j * sn[2]) / (8 * pi)
    assert abs(k - ev(SPEC["kernel"]["cases"][2]["value"])) < 2e-17
    for c in SPEC["chebyshev"]["cases"]:
        V, T = cube_mesh(c["a"], c["b"])
        t = pb.Tree(V, T, 10 ** 6, 1.0, c["m"])
        ex = t.export()
        assert ex["clusters"].shape[0] == 1
        assert np.array_equal(ex["boxes"][0], np.array([c["a"]] * 3 + [c["b"]] * 3, dtype=float))
