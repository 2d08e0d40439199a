"""Pins of the tcgen05 descriptor encodings the implicit convolution relies on
(row-shifted start addresses, LBO = 16 B pairing), against an exact host reference."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_06445_b200 import codedinv
    return codedinv


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
