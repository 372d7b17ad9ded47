"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports
every symbol include/bem.h declares, validates arguments, and its host-side
structure (frequencies, tree, partition) is bit-identical to the oracle's."""
import re
import os

import numpy as np
import pytest

import oracle as O
import synth
import paper_2006_05186_b200 as pb
from paper_2006_05186_b200 import bem as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "bem.h")).read()
    names = set(re.findall(r"^(?:bem_status|const char\*)\s+(\w+)\s*\(", hdr, flags=re.M))
    assert {"bem_build_tree", "bem_assemble_h2_aca", "bem_apply_multifreq", "cqm_forward", "cqm_inverse",
            "cqm_solve", "cqm_frequencies"} <= names
    lib = pb.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert names <= set(B.EXPORTS)


@pytest.mark.parametrize("N,T,method", [(1, 1.0, 2), (32, 2.0, 2), (128, 2.0, 2), (257, 2.0, 2), (64, 3.0, 1)])
def test_frequencies_bit_identical_to_oracle(N, T, method):
    """C14: the oracle's s_l and the library's are bit-equal (same host libm)."""
    R = 10.0 ** (-5.0 / N) if N > 1 else 1e-5
    a = pb.cqm_frequencies(N, T, R, method)
    b = O.frequencies(N, T, R, method)
    assert np.array_equal(a.view(np.float64), b.view(np.float64))


def test_argument_validation():
    with pytest.raises(B.BemError) as e:
        pb.cqm_frequencies(0, 2.0)
    assert e.value.code == -1
    with pytest.raises(B.BemError):
        pb.cqm_frequencies(8, 2.0, R=1.5)
    V, T = synth.icosphere(1)
    with pytest.raises(B.BemError):
        pb.Tree(V, T, 1, 1.0, 2, device=-1)  # leaf_size must be > 1
    with pytest.raises(B.BemError):
        pb.Tree(V, T, 8, 0.0, 2, device=-1)  # eta > 0
    with pytest.raises(B.BemError):
        pb.Tree(V, T, 8, 1.0, 0, device=-1)  # m >= 1
    bad = T.copy()
    bad[3, 1] = len(V) + 5
    with pytest.raises(B.BemError):
        pb.Tree(V, bad, 8, 1.0, 2, device=-1)
    deg = T.copy()
    deg[0] = [deg[0, 0], deg[0, 0], deg[0, 1]]
    with pytest.raises(B.BemError):
        pb.Tree(V, deg, 8, 1.0, 2, device=-1)
    t = pb.Tree(V, T, 8, 1.0, 2, device=-1)
    with pytest.raises(B.BemError) as e:
        pb.Operator(t, pb.cqm_frequencies(8, 2.0), 1e-6)
    assert e.value.code == -6  # host-only tree cannot carry an operator


def _tree_meshes():
    yield "cfg2", synth.icosphere(4), 32, 1.0, 3
    yield "cfg3", synth.ellipsoid(5), 48, 1.0, 4
    yield "sub3_eta2", synth.icosphere(3), 20, 2.0, 2
    yield "single", synth.icosphere(2), 10 ** 6, 1.0, 2
    V, T = synth.two_spheres(3, split=True)
    yield "two_split", (V, T), 24, 1.0, 3


@pytest.mark.parametrize("case", list(_tree_meshes()), ids=lambda c: c[0])
def test_tree_partition_bit_identical_to_oracle(case):
    """north_star: bit-exact cluster trees and admissibility lists (C13)."""
    _, (V, T), nmin, eta, m = case
    lt = pb.Tree(V, T, nmin, eta, m, device=-1)
    oh = O.H2(V, T, nmin, eta, m)
    a, b = lt.export(), oh.export()
    for k in ("perm", "clusters", "boxes", "near", "far"):
        assert a[k].shape == b[k].shape, k
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
    assert lt.stats["nnz_near"] == oh.nnz_near and lt.stats["depth"] == oh.depth


@pytest.mark.parametrize("cfg", [4, 5])
def test_tree_partition_full_size_bit_identical(cfg):
    """Configs 4 and 5 at full size (81,920 / 327,680 panels): the library's tree and
    partition (host build, the same code the device build runs) bit-equal to the oracle's."""
    c = synth.CONFIGS[cfg]
    V, T = synth.config_mesh(cfg)
    lt = pb.Tree(V, T, c["leaf"], c["eta"], c["m"], device=-1)
    oh = O.H2(V, T, c["leaf"], c["eta"], c["m"])
    a, b = lt.export(), oh.export()
    for k in ("perm", "clusters", "boxes", "near", "far"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_tree_cfg4_stats_match_probe():
    """SURVEY §8.0 row 4 (independent probe): 3,591 clusters, 1,796 leaves,
    63,554 near and 98,386 far blocks."""
    V, T = synth.icosphere(6)
    lt = pb.Tree(V, T, 64, 1.0, 4, device=-1)
    s = lt.stats
    assert (s["clusters"], s["leaves"], s["near_blocks"], s["far_blocks"]) == (3591, 1796, 63554, 98386)


def test_null_handles_rejected_without_gpu():
    """The newer entry points (combined mode, time-domain path, one-call step)
    validate their handles before touching a device: NULL -> BEM_EINVAL."""
    lib = pb.lib()
    assert lib.bem_aca_export_near(None, None, None, None) == -1
    assert lib.bem_mot_prepare(None, 0.5, None) == -1
    assert lib.bem_conv_time(None, None, None, 0, None) == -1
    assert lib.cqm_mot_solve(None, None, None, 1e-8, 10, 10, None, None) == -1
    assert lib.bem_time_step(None, None, None, 0.5, None) == -1
    assert lib.bem_op_get_info(None, None) == -1
    assert lib.bem_op_get_work(None, None) == -1
    assert b"NULL" in lib.bem_last_error()
