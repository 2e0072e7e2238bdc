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


def _shapes(seed, n):
    rng = np.random.default_rng(seed)
    return [tuple(int(8 * rng.integers(lo, hi)) for lo, hi in ((8, 90), (8, 120), (2, 80)))
            for _ in range(n)]


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", _shapes(11, 4))
def test_gemm_random_shapes(a_mn, b_mn, M, N, K):
    """Seeded random M / N / K (multiples of 8: TMA row pitch) for every
    operand-major form: partial M / N tiles and short or ragged K."""
    out, ref, _ = run_gemm(a_mn, b_mn, 1, M, N, K, seed=M + N + K)
    assert np.abs(out - ref).max() <= 1e-3 * np.sqrt(K), (M, N, K)


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (200, 328, 136), (1024, 1536, 512)])
def test_gemm_fused_adamw_epilogue(M, N, K):
    """Weight-gradient GEMM with the AdamW update in the epilogue (256-bit
    optimizer-state accesses, partial tiles): first step from m = v = 0 with
    lr 1e-3, betas (0.9, 0.95), no decay -> p - lr / (1 - 0.9) * m / (sqrt(v) / sqrt(1 - 0.95) + eps)."""
    rng = np.random.default_rng(M)
    A_bits, A = rand_bf16(rng, (M, K))
    B_bits, B = rand_bf16(rng, (N, K))
    A_st = np.ascontiguousarray(A_bits.T)  # MN-major, as the dW GEMMs
    B_st = np.ascontiguousarray(B_bits.T)
    p0 = (0.02 * rng.standard_normal((M, N))).astype(np.float32)
    Cbuf = p0.copy()
    ms = C.c_float(0)
    _lib.call("specsim_debug_gemm", 1, 1, 6 | (2 << 8), M, N, K, _lib.ptr(A_st), M,
              _lib.ptr(B_st), N, _lib.ptr(Cbuf), N, None, 0, 0, C.byref(ms))
    g = (A.astype(np.float64) @ B.astype(np.float64).T).astype(np.float32)
    m = 0.1 * g
    v = 0.05 * g * g
    ref = p0 - (1e-3 / 0.1) * m / (np.sqrt(v) / np.sqrt(0.05) + 1e-8)
    well = np.abs(g) > 1e-3 * np.abs(g).max()
    assert np.abs(Cbuf - ref)[well].max() <= 2e-5, np.abs(Cbuf - ref)[well].max()


def test_gemm_reduced_grid_is_exact():
    """SPECSIM_GEMM_SMS caps the persistent grid (SMs left to concurrent NCCL
    kernels in data-parallel runs); the tile loop must give identical results."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
            "import numpy as np; from test_gemm_gpu import run_gemm;"
            "o, r, _ = run_gemm(1, 1, 1, 2048, 1536, 512, seed=9);"
            "np.save('/tmp/specsim_gemm_grid.npy', o)")
    import os
    import pathlib
    root = pathlib.Path(__file__).resolve().parents[1]
    outs = []
    for sms in ("0", "40"):
        env = dict(os.environ, SPECSIM_GEMM_SMS=sms)
        subprocess.run([sys.executable, "-c", code], cwd=root, env=env, check=True)
        outs.append(np.load("/tmp/specsim_gemm_grid.npy"))
    assert np.array_equal(outs[0], outs[1])
