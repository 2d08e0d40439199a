"""Pins of the tcgen05 descriptor encodings the implicit convolution relies on
(row-shifted start addresses, LBO = 16 B pairing, fp16 operand type), against an exact host
reference, through the test-only probe library (include/codedinv_probe.h)."""
import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
PROBE_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2106_06445_b200",
                         "libcodedinv_probe.so")


class _Probe:
    """ctypes marshalling of libcodedinv_probe.so (test-only library)."""

    def __init__(self):
        self.lib = ctypes.CDLL(PROBE_LIB)
        P, I32 = ctypes.c_void_p, ctypes.c_int32
        self.lib.ci_probe_last_error.restype = ctypes.c_char_p
        self.lib.ci_test_umma_gemm.restype = I32
        self.lib.ci_test_umma_gemm.argtypes = [P, I32, I32, P, I32, I32, I32, I32, I32, P, P]
        self.lib.ci_test_umma_rate.restype = I32
        self.lib.ci_test_umma_rate.argtypes = [I32, I32, I32, P, P]

    def _check(self, st, where):
        if st != 0:
            raise RuntimeError(f"{where}: status {st}: {self.lib.ci_probe_last_error().decode()}")

    @staticmethod
    def _s():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def ci_test_umma_gemm(self, A, B, N, shift, mode, nk, D):
        self._check(self.lib.ci_test_umma_gemm(A.data_ptr(), A.shape[0], A.shape[1], B.data_ptr(), N, B.shape[1],
                                               shift, mode, nk, D.data_ptr(), self._s()), "ci_test_umma_gemm")

    def ci_test_umma_rate(self, N, iters, nblocks, cycles):
        self._check(self.lib.ci_test_umma_rate(N, iters, nblocks, cycles.data_ptr(), self._s()), "ci_test_umma_rate")


@pytest.fixture(scope="module")
def ci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _Probe()


def bf16_small_ints(rng, shape):
    # small integers are exact in bf16 and their products/sums exact in fp32
    return rng.integers(-8, 9, size=shape).astype(np.float32)


def to_bf16_bits(a):
    return torch.from_numpy(a).to(torch.bfloat16).view(torch.int16).cuda()


@pytest.mark.parametrize("N", [16, 32, 64, 96, 256])
@pytest.mark.parametrize("shift", [0, 1, 5, 17, 33])
def test_umma_gemm_row_shift(ci, N, shift):
    rng = np.random.default_rng(N * 100 + shift)
    nk, KA = 3, 48
    RA = 128 + shift + 8
    A = bf16_small_ints(rng, (RA, KA))
    B = bf16_small_ints(rng, (N, KA))
    D = torch.empty(128, N, device="cuda")
    ci.ci_test_umma_gemm(to_bf16_bits(A), to_bf16_bits(B), N, shift, 0, nk, D)
    torch.cuda.synchronize()
    ref = A[shift:shift + 128] @ B.T
    assert np.array_equal(D.cpu().numpy(), ref)


@pytest.mark.parametrize("shift", [0, 3, 18])
def test_umma_gemm_lbo16_pairs_adjacent_rows(ci, shift):
    rng = np.random.default_rng(shift)
    N, nk = 64, 3
    RA = 128 + shift + 2 * nk + 8
    A = bf16_small_ints(rng, (RA, 8))
    B = bf16_small_ints(rng, (N, 16 * nk))
    D = torch.empty(128, N, device="cuda")
    ci.ci_test_umma_gemm(to_bf16_bits(A), to_bf16_bits(B), N, shift, 1, nk, D)
    torch.cuda.synchronize()
    ref = np.zeros((128, N), np.float32)
    for j in range(nk):
        r0 = shift + 2 * j
        ref += A[r0:r0 + 128] @ B[:, 16 * j:16 * j + 8].T
        ref += A[r0 + 1:r0 + 129] @ B[:, 16 * j + 8:16 * j + 16].T
    assert np.array_equal(D.cpu().numpy(), ref)


@pytest.mark.parametrize("lbo_rows,shift", [(17, 0), (9, 4), (5, 2), (1187, 3), (300, 130)])
def test_umma_gemm_any_lbo(ci, lbo_rows, shift):
    """Any LBO is legal for K-major no-swizzle: the pair-mode vertical taps (LBO = Wp rows:
    17 / 9 / 5) and the tri mode's cross-plane pair (LBO = plane - (Wp+1) rows, here into the
    next plane: K-half 1 reads plane 1)."""
    rng = np.random.default_rng(lbo_rows * 7 + shift)
    N, nk, KA = 48, 3, 16
    RA = 1200 if lbo_rows > 200 else 160 + shift + lbo_rows
    A = bf16_small_ints(rng, (RA, KA))
    B = bf16_small_ints(rng, (N, 16 * nk))
    D = torch.empty(128, N, device="cuda")
    ci.ci_test_umma_gemm(to_bf16_bits(A), to_bf16_bits(B), N, shift, 2 | (lbo_rows << 8), nk, D)
    torch.cuda.synchronize()
    lin = np.concatenate([A[:, 0:8], A[:, 8:16]], axis=0)   # plane p row r -> row p*RA + r
    ref = np.zeros((128, N), np.float32)
    for j in range(nk):
        r0 = shift + j
        ref += lin[r0:r0 + 128] @ B[:, 16 * j:16 * j + 8].T
        ref += lin[r0 + lbo_rows:r0 + lbo_rows + 128] @ B[:, 16 * j + 8:16 * j + 16].T
    assert np.array_equal(D.cpu().numpy(), ref)


@pytest.mark.parametrize("N", [32, 128, 256])
def test_umma_gemm_fp16_operands(ci, N):
    """The f16x2 precision's instruction descriptor (a/b_format = F16): values j/512 with
    |j| < 1024 are exact in fp16 but not in bf16, and one K=16 step sums exactly in fp32."""
    rng = np.random.default_rng(N)
    RA, KA, nk, shift = 160, 16, 1, 7
    A = (rng.integers(-1023, 1024, size=(RA, KA)) / 512.0).astype(np.float32)
    B = (rng.integers(-1023, 1024, size=(N, KA)) / 512.0).astype(np.float32)
    D = torch.empty(128, N, device="cuda")
    to16 = lambda a: torch.from_numpy(a).to(torch.float16).view(torch.int16).cuda()
    ci.ci_test_umma_gemm(to16(A), to16(B), N, shift, 0 | (1 << 30), nk, D)
    torch.cuda.synchronize()
    ref = A[shift:shift + 128].astype(np.float64) @ B.T.astype(np.float64)
    assert np.array_equal(D.cpu().numpy().astype(np.float64), ref)


def test_umma_issue_rate_report(ci):
    """Reports the SS-mode tcgen05 rate (cycles per 128xNx16 MMA, 148 CTAs, tight issue loop;
    profiles/r01_umma_probe.md); sanity only."""
    for N in (16, 32, 64, 96, 128, 256):
        cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
        ci.ci_test_umma_rate(N, 2048, 148, cyc)
        torch.cuda.synchronize()
        c = cyc.cpu().numpy().astype(np.float64).mean() / 2048
        print(f"[umma rate] N={N}: {c:.1f} cyc/MMA (compute floor N/2 = {N / 2:.0f}, "
              f"SS model max(N/2, 32+N/4) = {max(N / 2, 32 + N / 4):.0f})")
        assert c >= N / 2 * 0.95


def _ts_probe(ci):
    P, I32 = ctypes.c_void_p, ctypes.c_int32
    ci.lib.ci_test_umma_ts_gemm.restype = I32
    ci.lib.ci_test_umma_ts_gemm.argtypes = [P, P, I32, I32, I32, I32, P, P]
    ci.lib.ci_test_umma_ts_rate.restype = I32
    ci.lib.ci_test_umma_ts_rate.argtypes = [I32, I32, I32, P, P]
    return ci.lib


@pytest.mark.parametrize("N,nk,acol", [(16, 1, 256), (80, 4, 256), (96, 2, 128), (128, 4, 384), (256, 3, 256)])
@pytest.mark.parametrize("f16", [0, 1])
def test_umma_ts_gemm_a_in_tmem(ci, N, nk, acol, f16):
    """TS mode (A operand in tensor memory, the stage-1 conv2 of DESIGN.md 7.2): lane r = row r,
    K pairs (2i, 2i+1) packed low / high in column 8j + i; exact on small integers."""
    lib = _ts_probe(ci)
    rng = np.random.default_rng(N * 10 + nk + f16)
    A = bf16_small_ints(rng, (128, 16 * nk))
    B = bf16_small_ints(rng, (N, 16 * nk))
    dt = torch.float16 if f16 else torch.bfloat16
    a16 = torch.from_numpy(A).to(dt).view(torch.int16).view(torch.int32).cuda()   # pairs -> one word, even k low
    b16 = torch.from_numpy(B).to(dt).view(torch.int16).cuda()
    D = torch.empty(128, N, device="cuda")
    st = lib.ci_test_umma_ts_gemm(a16.data_ptr(), b16.data_ptr(), N, nk, acol, f16, D.data_ptr(), ci._s())
    assert st == 0, ci.lib.ci_probe_last_error().decode()
    torch.cuda.synchronize()
    assert np.array_equal(D.cpu().numpy(), A @ B.T)


def test_umma_ts_issue_rate_report(ci):
    """Reports the TS-mode tcgen05 rate (A from TMEM: only B crosses the shared-memory port); sanity only."""
    lib = _ts_probe(ci)
    for N in (16, 32, 48, 64, 80, 96, 128, 160, 256):
        cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
        st = lib.ci_test_umma_ts_rate(N, 2048, 148, cyc.data_ptr(), ci._s())
        assert st == 0
        torch.cuda.synchronize()
        c = cyc.cpu().numpy().astype(np.float64).mean() / 2048
        print(f"[umma ts rate] N={N}: {c:.1f} cyc/MMA (compute floor N/2 = {N / 2:.0f}, "
              f"SS model max(N/2, 32+N/4) = {max(N / 2, 32 + N / 4):.0f})")
        assert c >= N / 2 * 0.95
