"""The tcgen05 kind::i8 layout conventions the INT8 coupling kernel (far10) relies
on: D = A B^T from the tensor cores (A in tensor memory or shared memory, B in the
K-major canonical shared-memory layout, D read back from tensor memory) equals the
plain integer product, bit for bit."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("K,N", [(32, 64), (128, 64), (256, 128), (512, 16)])
def test_i8_gemm_matches_integer_product(mode, K, N):
    import paper_2006_05186_b200 as pb
    from paper_2006_05186_b200.bem import _check, lib
    rng = np.random.default_rng(K * 7 + N + mode)
    A = rng.integers(-128, 128, (128, K), dtype=np.int8)
    B = rng.integers(-128, 128, (N, K), dtype=np.int8)
    D = np.zeros((128, N), dtype=np.int32)
    _check(lib().bem_debug_i8_gemm(A.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                                   D.ctypes.data_as(C.c_void_p), K, N, mode, 0))
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(D.astype(np.int64), ref)


@pytest.mark.parametrize("K,N", [(32, 64), (128, 64), (256, 128)])
def test_i8_gemm_pair_matches_integer_product(K, N):
    """cta_group::2 (M = 256 over two CTAs): CTA r holds A rows 128 r.. and B rows r N/2.."""
    from paper_2006_05186_b200.bem import _check, lib
    rng = np.random.default_rng(K * 3 + N)
    A = rng.integers(-128, 128, (256, K), dtype=np.int8)
    B = rng.integers(-128, 128, (N, K), dtype=np.int8)
    D = np.zeros((256, N), dtype=np.int32)
    _check(lib().bem_debug_i8_gemm_pair(A.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                                        D.ctypes.data_as(C.c_void_p), K, N, 0))
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(D.astype(np.int64), ref)
