"""GPU parity of the i-ResNet variant.

Residual blocks y = x + G(x), G = conv3x3 -> ELU -> conv3x3 on the whole state, weights
spectrally normalised to Lip(G) <= 0.9 (fixtures); h^-1 runs arch.fp_iters = 10 fixed-point
updates x <- y - G(x) per block.  The GPU is compared with the oracle run for the SAME number
of updates (isolates arithmetic precision) and with the oracle's converged inverse (adds the
truncation of the fixed point, ~3e-7 at L = 0.9, N = 10).  Tolerances as in
test_gpu_parity.py: 1e-3 (fp32: f16x3 products for residual archs), 3e-2 (bf16, reported).
"""
import numpy as np
import pytest

import fixtures as fx
import oracle

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


def relerr(a, ref):
    a = np.asarray(a, np.float64).reshape(-1, np.shape(ref)[-1])
    r = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


def h_and_inverse(ci, arch, params, prec, x):
    n = x.shape[0]
    m = ci.Model(arch, params, prec)
    ws = m.workspace(1, n)
    h = torch.empty(n, arch.d, device="cuda")
    m.ci_forward_h(dev(x), h, ws)
    href = oracle.forward_h(arch, params, x)
    xr = torch.empty(n, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    m.ci_inverse_h(dev(href.astype(np.float32)), xr, ws)       # invert the oracle's h
    xrt = torch.empty_like(xr)
    m.ci_inverse_h(h, xrt, ws)                                  # GPU round trip
    torch.cuda.synchronize()
    return h.cpu().numpy(), href, xr.cpu().numpy(), xrt.cpu().numpy()


@pytest.mark.parametrize("prec", PRECS)
def test_residual_h_and_fixed_point_inverse_small(ci, prec):
    """Arch TR, 37 images (several 128-row tiles and a ragged tail)."""
    arch = fx.ARCH_TR
    params = fx.make_weights(arch, 5)
    x = fx.make_inputs(arch, 1, 37, 2)[0]
    h, href, xr, xrt = h_and_inverse(ci, arch, params, prec, x)
    e_h = relerr(h, href)
    same_n = oracle.inverse_h(arch, params, href.astype(np.float32), fp_iters=arch.fp_iters)
    conv = oracle.inverse_h(arch, params, href.astype(np.float32))
    e_inv = relerr(xr.reshape(37, -1), same_n.reshape(37, -1))
    e_conv = relerr(xr.reshape(37, -1), conv.reshape(37, -1))
    e_rt = relerr(xrt.reshape(37, -1), x.reshape(37, -1))
    print(f"[TR {prec}] h={e_h:.3g} inv(N={arch.fp_iters})={e_inv:.3g} inv(converged)={e_conv:.3g} "
          f"round-trip={e_rt:.3g}")
    tol = TOL[prec]
    assert e_h < tol and e_inv < tol and e_conv < tol and e_rt < tol


@pytest.mark.parametrize("prec", PRECS)
def test_residual_serve_small(ci, prec):
    """Whole coded path on Arch TR (exact encode = fixed-point h^-1 of the mean)."""
    arch = fx.ARCH_TR
    B, k = 5, 3
    params = fx.make_weights(arch, 6)
    x, drop = fx.make_inputs(arch, B, k, 4), fx.make_drops(B, k, 9)
    ref = oracle.serve_group(arch, params, x, drop, fp_iters=arch.fp_iters)
    m = ci.Model(arch, params, prec)
    h = torch.empty(B, k, arch.d, device="cuda")
    p = torch.empty(B, arch.d, device="cuda")
    xp = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    logits = torch.empty(B * k * 10, device="cuda")
    labels = torch.empty(B * k, dtype=torch.int32, device="cuda")
    ws = m.workspace(k, B)
    m.ci_serve_group(dev(x), dev(drop), h, p, ws, x_parity=xp, logits=logits, labels=labels)
    m.ci_check(ws)
    e = dict(R=relerr(h.cpu().numpy(), ref["R"]), P=relerr(p.cpu().numpy(), ref["P"]),
             xp=relerr(xp.cpu().numpy().reshape(B, -1), ref["xp"].reshape(B, -1)),
             logits=relerr(logits.cpu().numpy().reshape(B, k, 10), ref["logits"][0]))
    print(f"[TR serve {prec}] " + " ".join(f"{a}={b:.3g}" for a, b in e.items()))
    assert max(e.values()) < TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_residual_arch_c_sampled(ci, prec):
    """Arch CR (channel plan 12/48/192, m = 64/128/256): 1024 images through h and h^-1 at
    once (the tcgen05 launch size of a C3-like batch), 3 sampled images checked one by one."""
    arch = fx.ARCH_CR
    params = fx.make_weights(arch, 13)
    n = 1024
    x = fx.make_inputs(arch, 1, n, 3)[0]
    m = ci.Model(arch, params, prec)
    ws = m.workspace(1, n)
    h = torch.empty(n, arch.d, device="cuda")
    m.ci_forward_h(dev(x), h, ws)
    xr = torch.empty(n, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    m.ci_inverse_h(h, xr, ws)
    torch.cuda.synchronize()
    sample = np.array([0, 517, n - 1])
    href = oracle.forward_h(arch, params, x[sample])
    e_h = relerr(h.cpu().numpy()[sample], href)
    xs = oracle.inverse_h(arch, params, h.cpu().numpy()[sample], fp_iters=arch.fp_iters)
    e_inv = relerr(xr.cpu().numpy()[sample].reshape(3, -1), xs.reshape(3, -1))
    e_rt = relerr(xr.cpu().numpy().reshape(n, -1), x.reshape(n, -1))
    print(f"[CR {prec}] h={e_h:.3g} inv(N={arch.fp_iters})={e_inv:.3g} round-trip(all {n})={e_rt:.3g}")
    tol = TOL[prec]
    assert e_h < tol and e_inv < tol and e_rt < tol
