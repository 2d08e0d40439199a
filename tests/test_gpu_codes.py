"""GPU parity of general (n, k) codes against the
f64 oracle (oracle/codes.py).  Both sides use the same fp32 coefficients (promoted exactly on
the oracle side).  Decoding from a subset S amplifies upstream feature errors by at most
||inv(G_S)||_inf, so tolerances are TOL[prec] x that amplification (printed)."""
import itertools

import numpy as np
import pytest

import fixtures as fx
import oracle
from oracle import codes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PRECS = ["fp32", "f16x2", "bf16"]
TOL = {"fp32": 1e-3, "f16x2": 5e-3, "bf16": 3e-2}


@pytest.fixture(scope="module")
def ci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_06445_b200 import codedinv
    return codedinv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gen32(n, k, scheme, seed=1):
    """(fp32 parity rows for the GPU, the same generator in f64 for the oracle)"""
    G = codes.build_generator(n, k, scheme, seed=seed)
    c32 = G[k:].astype(np.float32)
    G64 = G.copy()
    G64[k:] = c32.astype(np.float64)
    return c32, G64


def amplification(G, avail, k):
    return max(np.abs(codes.subset_inverse(G, codes.decode_subset(int(a), G.shape[0], k))).sum(1).max()
               for a in avail)


def relerr_rows(a, ref):
    a = np.asarray(a, np.float64).reshape(-1, ref.shape[-1])
    r = np.asarray(ref, np.float64).reshape(-1, ref.shape[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


@pytest.mark.parametrize("n,k,scheme", [(4, 2, "paper42"), (6, 4, "vandermonde"), (7, 3, "gaussian"),
                                        (11, 10, "uniform"), (20, 16, "gaussian")])
def test_decode_general_vs_oracle(ci, n, k, scheme):
    c32, G = gen32(n, k, scheme)
    r = n - k
    rng = np.random.default_rng(n * 31 + k)
    B, d = 97, 3072
    F = rng.standard_normal((B, k, d))                       # true f(x_1..k)
    P = np.einsum("ij,bjd->bid", G[k:], F)                   # ideal parity results
    # availability: every group loses a random number (0..r) of tasks, at least k remain
    avail = np.zeros(B, np.uint32)
    for b in range(B):
        lost = rng.choice(n, size=rng.integers(0, r + 1), replace=False)
        avail[b] = sum(1 << t for t in range(n) if t not in lost)
    Hin = F.astype(np.float32)
    Hin_lost = Hin.copy()
    for b in range(B):
        for j in range(k):
            if not (avail[b] >> j) & 1:
                Hin_lost[b, j] = np.nan                      # must be overwritten
    Ht = dev(Hin_lost)
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    ci.ci_decode_general(dev(c32), Ht, dev(P.astype(np.float32)), dev(avail.view(np.int32)), ws)
    got = Ht.cpu().numpy()
    ref = codes.decode(G, np.concatenate([Hin.astype(np.float64), P.astype(np.float32).astype(np.float64)], 1),
                       avail)
    amp = amplification(G, avail, k)
    e = relerr_rows(got, ref)
    print(f"[decode_general ({n},{k}) {scheme}] err={e:.3g} amplification={amp:.3g}")
    assert not np.isnan(got).any()
    assert e < 1e-6 * amp
    # available main tasks are untouched (bit-exact)
    for b in range(B):
        for j in range(k):
            if (avail[b] >> j) & 1:
                assert np.array_equal(got[b, j], Hin[b, j])


def test_decode_general_uniform_equals_hot_path_decode(ci):
    k, B, d = 10, 64, 3072
    c32, G = gen32(k + 1, k, "uniform")
    rng = np.random.default_rng(2)
    H = rng.standard_normal((B, k, d)).astype(np.float32)
    P = H.mean(1).astype(np.float32)
    drop = rng.integers(0, k, B).astype(np.int32)
    avail = np.array([((1 << (k + 1)) - 1) & ~(1 << int(j)) for j in drop], np.uint32)
    a, b_ = dev(H), dev(H)
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    ci.ci_decode_general(dev(c32), a, dev(P), dev(avail.view(np.int32)), ws)
    ci.ci_decode(b_, dev(P), dev(drop), ws)
    assert relerr_rows(a.cpu().numpy(), b_.cpu().numpy().astype(np.float64)) < 2e-6


def test_decode_general_flags_undecodable(ci):
    c32, G = gen32(4, 2, "paper42")
    H = np.ones((3, 2, 8), np.float32)
    Pp = np.ones((3, 2, 8), np.float32)
    avail = np.array([0b1111, 0b1000, 0b0100], np.uint32)    # groups 1, 2: one result only
    Ht = dev(H)
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    ci.ci_decode_general(dev(c32), Ht, dev(Pp), dev(avail.view(np.int32)), ws)
    torch.cuda.synchronize()
    assert int(ws[4:8].view(torch.int32).item()) == 2          # the undecodable count (flag int 1)
    assert np.array_equal(Ht.cpu().numpy(), H)
    with pytest.raises(ci.CiError) as e:
        ci._check(ci._lib.ci_check(None, ci._ptr(ws), ws.numel(), ci._stream(None)), "ci_check")
    assert e.value.status == ci.CI_ERR_UNDECODABLE


@pytest.mark.parametrize("scale", [1.0, 1e-14])
def test_decode_general_singular_subset_is_scale_invariant(ci, scale):
    """A non-MDS code (SPEC.md:59 SingularSubset): parity rows [a, 2a] and [a, 2a(1 + 1e-12)]
    (= [a, 2a] in fp32) with both mains lost leave a singular subset: left untouched and flagged,
    whatever the scale a.  An invertible pair of rows [a, 2a], [2a, a] decodes at any scale (at
    a = 1e-14 an absolute pivot floor of 1e-12 would have called it singular; the row-normalised
    determinant is 3/5)."""
    k, d = 2, 8
    a = scale
    coef = np.array([[a, 2 * a], [a, 2 * a + 1e-12 * a]], np.float32)
    coef_ok = np.array([[a, 2 * a], [2 * a, a]], np.float32)
    F = np.array([[1.0, -2.0], [0.5, 3.0]])                          # true f(x_1), f(x_2) of 2 groups
    Fd = np.repeat(F[:, :, None], d, axis=2).astype(np.float32)       # [B=2][k][d]
    for c, singular in ((coef, True), (coef_ok, False)):
        P = np.einsum("rk,bkd->brd", c.astype(np.float64), Fd.astype(np.float64)).astype(np.float32)
        Ht = dev(np.zeros_like(Fd))
        avail = np.array([0b1100, 0b1100], np.uint32)                 # only the two parities arrived
        ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
        ci.ci_decode_general(dev(c), Ht, dev(P), dev(avail.view(np.int32)), ws)
        torch.cuda.synchronize()
        got = Ht.cpu().numpy()
        if singular:
            assert int(ws[4:8].view(torch.int32).item()) == 2 and np.all(got == 0)
        else:
            assert int(ws[4:8].view(torch.int32).item()) == 0
            assert np.max(np.abs(got - Fd)) < 1e-5


def run_serve_general(ci, m, arch, c32, x, avail):
    B, k = x.shape[:2]
    r = c32.shape[0]
    h = torch.empty(B, k, arch.d, device="cuda")
    hp = torch.empty(B, r, arch.d, device="cuda")
    xp = torch.empty(B, r, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    logits = torch.empty(B * k * 10, device="cuda")
    labels = torch.empty(B * k, dtype=torch.int32, device="cuda")
    ws = m.workspace_general(k, r, B)
    m.ci_serve_general(dev(c32), dev(x), dev(avail.view(np.int32)), h, hp, ws, x_parity=xp, logits=logits,
                       labels=labels)
    m.ci_check(ws)
    return dict(R=h.cpu().numpy(), P=hp.cpu().numpy(), xp=xp.cpu().numpy(),
                logits=logits.cpu().numpy().reshape(B, k, 10), labels=labels.cpu().numpy().reshape(B, k))


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("arch_name,n,k,scheme", [("T", 4, 2, "paper42"), ("M", 6, 4, "vandermonde"),
                                                  ("TR", 4, 2, "paper42")])
def test_serve_general_every_subset(ci, prec, arch_name, n, k, scheme):
    """Every k-subset of tasks as the available set (PAPER.md:591 'any two of the four')."""
    arch = fx.ARCHS[arch_name]
    params = fx.make_weights(arch, 4)
    c32, G = gen32(n, k, scheme)
    subsets = list(itertools.combinations(range(n), k)) + [tuple(range(n))]
    B = len(subsets)
    avail = np.array([sum(1 << t for t in S) for S in subsets], np.uint32)
    x = fx.make_inputs(arch, B, k, 8)
    ref = codes.serve_general(arch, params, x, G, avail, fp_iters=arch.fp_iters)
    g = run_serve_general(ci, ci.Model(arch, params, prec), arch, c32, x, avail)
    amp = amplification(G, avail, k)
    e = dict(R=relerr_rows(g["R"], ref["R"]), P=relerr_rows(g["P"], ref["P"]),
             xp=relerr_rows(g["xp"].reshape(B * (n - k), -1), ref["xp"].reshape(B * (n - k), -1)),
             logits=relerr_rows(g["logits"], ref["logits"][0]))
    print(f"[serve_general {arch_name} ({n},{k}) {scheme} {prec}] amp={amp:.3g} " +
          " ".join(f"{a}={b:.3g}" for a, b in e.items()))
    tol = TOL[prec]
    assert e["P"] < tol and e["xp"] < tol
    assert e["R"] < tol * amp and e["logits"] < tol * amp


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_serve_general_arch_c_sampled(ci, prec):
    """Arch C, (12, 10) Vandermonde code (two parity queries per group), 1024 groups each
    losing two random tasks; 3 groups checked against the oracle."""
    arch, k, n, B = fx.ARCH_C, 10, 12, 1024
    params = fx.make_weights(arch, 13)
    c32, G = gen32(n, k, "vandermonde")
    rng = np.random.default_rng(5)
    avail = np.array([((1 << n) - 1) & ~sum(1 << int(t) for t in rng.choice(n, 2, replace=False))
                      for _ in range(B)], np.uint32)
    x = fx.make_inputs(arch, B, k, 3)
    g = run_serve_general(ci, ci.Model(arch, params, prec), arch, c32, x, avail)
    sample = np.array([0, 511, B - 1])
    ref = codes.serve_general(arch, params, x[sample], G, avail[sample])
    amp = amplification(G, avail[sample], k)
    e = dict(R=relerr_rows(g["R"][sample], ref["R"]), P=relerr_rows(g["P"][sample], ref["P"]),
             logits=relerr_rows(g["logits"][sample], ref["logits"][0]))
    print(f"[serve_general C (12,10) {prec}] amp={amp:.3g} " + " ".join(f"{a}={b:.3g}" for a, b in e.items()))
    tol = TOL[prec]
    assert e["P"] < tol and e["R"] < tol * amp and e["logits"] < tol * amp


@pytest.mark.parametrize("prec", PRECS)
def test_perturbed_encode_and_k_eps_law(ci, prec):
    """f4: x_p = h^-1(mean + eps) on the GPU vs the oracle; eps = 0 reproduces ci_encode bit for
    bit; decoding the perturbed parity returns f(x_a) + k eps."""
    arch = fx.ARCH_M
    k, B = 4, 64
    params = fx.make_weights(arch, 2)
    x = fx.make_inputs(arch, B, k, 6)
    m = ci.Model(arch, params, prec)
    ws = m.workspace(k, B)
    h = torch.empty(B, k, arch.d, device="cuda")
    m.ci_forward_h(dev(x.reshape(B * k, *x.shape[2:])), h.view(B * k, arch.d), ws)
    xp0 = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    xpz = torch.empty_like(xp0)
    m.ci_encode(h, xp0, ws)
    m.ci_encode_perturbed(h, torch.zeros(B, arch.d, device="cuda"), xpz, ws)
    torch.cuda.synchronize()
    assert torch.equal(xp0, xpz)
    eps = (1e-2 * np.random.default_rng(3).standard_normal((B, arch.d))).astype(np.float32)
    xp = torch.empty_like(xp0)
    m.ci_encode_perturbed(h, dev(eps), xp, ws)
    _, xref = oracle.encode_perturbed(arch, params, h.cpu().numpy().astype(np.float64), eps)
    e_xp = relerr_rows(xp.cpu().numpy().reshape(B, -1), xref.reshape(B, -1))
    P = torch.empty(B, arch.d, device="cuda")
    m.ci_forward_h(xp, P, ws)
    drop = (np.arange(B) % k).astype(np.int32)
    R = h.clone()
    ci.ci_decode(R, P, dev(drop), ws)
    torch.cuda.synchronize()
    Hn, Rn = h.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    err = Rn[np.arange(B), drop] - Hn[np.arange(B), drop]
    law = np.max(np.abs(err - k * eps)) / np.max(np.abs(k * eps))
    print(f"[perturbed {prec}] xp={e_xp:.3g} k-eps-law residual={law:.3g}")
    assert e_xp < TOL[prec]
    assert law < (2e-2 if prec != "bf16" else 1.0)
