"""tcgen05 GEMM parity: every operand-major form and epilogue vs a float64
numpy product of the same bf16 inputs (fp32 accumulation tolerance)."""
import ctypes as C

import numpy as np
import pytest

from paper_2602_05145_b200 import _lib
from _util import rand_bf16, bf16_bits_to_f32

pytestmark = pytest.mark.gpu


def run_gemm(a_mn, b_mn, epi, M, N, K, seed=0, iters=0, cg=2):
    rng = np.random.default_rng(seed)
    # logical A [M,K], B [N,K]; stored per major-ness
    A_bits, A = rand_bf16(rng, (M, K))
    B_bits, B = rand_bf16(rng, (N, K))
    A_st = np.ascontiguousarray(A_bits.T) if a_mn else A_bits
    B_st = np.ascontiguousarray(B_bits.T) if b_mn else B_bits
    lda = A_st.shape[1]
    ldb = B_st.shape[1]
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    R_bits = None
    if epi in (1, 2):
        Cbuf = rng.standard_normal((M, N)).astype(np.float32) if epi == 2 else np.zeros((M, N), np.float32)
        if epi == 2:
            ref = ref + Cbuf.astype(np.float64)
    else:
        Cbuf = np.zeros((M, N), np.uint16)
    if epi == 3:
        R_bits, R = rand_bf16(rng, (M, N))
        ref = ref + R.astype(np.float64)
    ms = C.c_float(0)
    _lib.call("specsim_debug_gemm", a_mn, b_mn, epi | (cg << 8), M, N, K, _lib.ptr(A_st), lda, _lib.ptr(B_st),
              ldb, _lib.ptr(Cbuf), N, _lib.ptr(R_bits), N, iters, C.byref(ms))
    out = Cbuf if epi in (1, 2) else bf16_bits_to_f32(Cbuf)
    return out, ref, ms.value


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 320), (384, 768, 1024), (200, 328, 136)])
def test_gemm_forms_f32(a_mn, b_mn, M, N, K, cg):
    out, ref, _ = run_gemm(a_mn, b_mn, 1, M, N, K, cg=cg)
    err = np.abs(out - ref).max()
    assert err <= 1e-3 * np.sqrt(K), (err, out[:2, :4], ref[:2, :4])


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("epi", [0, 2, 3])
def test_gemm_epilogues(epi, cg):
    M, N, K = 256, 512, 256
    out, ref, _ = run_gemm(0, 0, epi, M, N, K, seed=3, cg=cg)
    if epi == 2:
        np.testing.assert_allclose(out, ref, atol=2e-3 * np.sqrt(K))
    else:  # bf16 output: one rounding of the fp32 result
        np.testing.assert_allclose(out, ref, rtol=1.0 / 128, atol=1e-2)


@pytest.mark.parametrize("cg", [1, 2])
def test_gemm_many_tiles_persistent(cg):
    # more tiles than SMs -> exercises the persistent loop, both TMEM stages and
    # the grouped rasterisation (several row groups)
    out, ref, _ = run_gemm(0, 0, 1, 2048, 4096, 256, seed=5, cg=cg)
    assert np.abs(out - ref).max() <= 1e-3 * 16
    out, ref, _ = run_gemm(1, 1, 1, 4096, 512, 2048, seed=6, cg=cg)
    assert np.abs(out - ref).max() <= 1e-3 * 46
