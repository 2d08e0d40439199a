"""The TS-mode stage kernels (csrc/k_stage_ts.cu stage 1, csrc/k_stage_ts2.cu stage 2; DESIGN.md
7.2b/c) against the f64 oracle and against the padded-raster k_stage (CI_NO_TS=1, CI_NO_TS2=1,
independently pinned by the round-1 tests).

Arch C's first two stages (16x16, c = 6, m = 64; 8x8, c = 24, m = 128) run on the TS kernels
whenever the model is created without those switches.  Image counts cover: one image (the pair's second slot absent), an odd count,
exactly one image per CTA pair, more images than 2 x 148 (dynamic claiming, two passes), and
the inverse direction (blocks in reverse order, subtraction)."""
import os

import numpy as np
import pytest

import fixtures as fx
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-3, "f16x2": 5e-3, "bf16": 3e-2}


@pytest.fixture(scope="module")
def ci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_06445_b200 import codedinv
    return codedinv


def relerr(a, ref):
    a = np.asarray(a, np.float64).reshape(-1, np.shape(ref)[-1])
    r = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


def make_model(ci, arch, params, prec, ts):
    """ts=False: both TS kernels off (CI_NO_TS, CI_NO_TS2: stages 1-2 on the padded k_stage)."""
    keys = ("CI_NO_TS", "CI_NO_TS2")
    old = {k: os.environ.pop(k, None) for k in keys}
    if not ts:
        for k in keys:
            os.environ[k] = "1"
    try:
        return ci.Model(arch, params, prec)
    finally:
        for k in keys:
            os.environ.pop(k, None)
            if old[k] is not None:
                os.environ[k] = old[k]


def run_h(m, x, n, d, inverse=False):
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ws = m.workspace(1, n)
    if inverse:
        out = torch.empty(n, 3, 32, 32, device="cuda")
        m.ci_inverse_h(xt.view(n, d), out, ws)
    else:
        out = torch.empty(n, d, device="cuda")
        m.ci_forward_h(xt.view(n, 3, 32, 32), out, ws)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(n, -1)


@pytest.mark.parametrize("prec", ["fp32", "f16x2", "bf16"])
@pytest.mark.parametrize("n", [1, 3, 296, 301])
def test_ts_forward_vs_oracle(ci, prec, n):
    arch = fx.ARCH_C
    params = fx.make_weights(arch, 13)
    x = fx.make_inputs(arch, 1, n, 7 + n)[0]
    got = run_h(make_model(ci, arch, params, prec, True), x, n, arch.d)
    idx = np.unique(np.array([0, n - 1, n // 2]))
    ref = oracle.forward_h(arch, params, x[idx]).reshape(len(idx), -1)
    e = relerr(got[idx], ref)
    print(f"[ts fwd {prec} n={n}] {e:.3g}")
    assert e < TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "f16x2"])
def test_ts_matches_padded_kernel(ci, prec):
    """Same h from the TS kernel and from the padded-raster k_stage (different MMA and epilogue
    order, same precision): agreement far inside the contract tolerance, forward and inverse."""
    arch = fx.ARCH_C
    params = fx.make_weights(arch, 13)
    n = 157
    x = fx.make_inputs(arch, 1, n, 99)[0]
    a = make_model(ci, arch, params, prec, True)
    b = make_model(ci, arch, params, prec, False)
    ha, hb = run_h(a, x, n, arch.d), run_h(b, x, n, arch.d)
    e_f = relerr(ha, hb)
    xa, xb = run_h(a, ha, n, arch.d, inverse=True), run_h(b, ha, n, arch.d, inverse=True)
    e_i = relerr(xa, xb)
    e_rt = relerr(xa, x.reshape(n, -1))
    print(f"[ts vs padded {prec}] forward {e_f:.3g} inverse {e_i:.3g} round trip {e_rt:.3g}")
    assert e_f < 1e-4 and e_i < 1e-4 and e_rt < 1e-5


def test_ts_inverse_vs_oracle_and_determinism(ci):
    arch = fx.ARCH_C
    params = fx.make_weights(arch, 13)
    n = 149
    x = fx.make_inputs(arch, 1, n, 5)[0]
    m = make_model(ci, arch, params, "fp32", True)
    h1 = run_h(m, x, n, arch.d)
    h2 = run_h(m, x, n, arch.d)
    assert np.array_equal(h1, h2)   # dynamic batch claiming does not change any result
    idx = np.array([0, 74, 148])
    ref = oracle.inverse_h(arch, params, h1[idx].astype(np.float64)).reshape(len(idx), -1)
    xr = run_h(m, h1, n, arch.d, inverse=True)
    e = relerr(xr[idx], ref)
    print(f"[ts inverse fp32] {e:.3g}")
    assert e < 1e-3


@pytest.mark.parametrize("k", [1, 10])
def test_ts_degenerate_single_group(ci, k):
    """One group through ci_serve_group on Arch C (the parity path is a single image: the TS
    kernels' second slot and the second image of a TS2 slot are absent; k = 1 is repetition, so
    x_p = x up to the round trip)."""
    arch = fx.ARCH_C
    params = fx.make_weights(arch, 13)
    x = fx.make_inputs(arch, 1, k, 21)
    drop = np.zeros(1, np.int32)
    ref = oracle.serve_group(arch, params, x, drop)
    m = make_model(ci, arch, params, "fp32", True)
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    h = torch.empty(1, k, arch.d, device="cuda")
    p = torch.empty(1, arch.d, device="cuda")
    xp = torch.empty(1, arch.in_c, arch.in_h, arch.in_w, device="cuda")
    ws = m.workspace(k, 1)
    m.ci_serve_group(xt, torch.from_numpy(drop).cuda(), h, p, ws, x_parity=xp)
    m.ci_check(ws)
    torch.cuda.synchronize()
    e = {key: relerr(g, ref[key]) for key, g in (("R", h.cpu().numpy()), ("P", p.cpu().numpy()),
                                                 ("xp", xp.cpu().numpy()))}
    print(f"[ts single group k={k}] " + " ".join(f"{a}={b:.3g}" for a, b in e.items()))
    assert max(e.values()) < 1e-3
    if k == 1:
        assert relerr(xp.cpu().numpy().reshape(1, -1), x.reshape(1, -1)) < 1e-5


_MC_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
arch = fx.ARCH_C
m = ci.Model(arch, fx.make_weights(arch, 13), sys.argv[2])
n = int(sys.argv[3])
x = torch.from_numpy(np.ascontiguousarray(fx.make_inputs(arch, 1, n, 41)[0])).cuda()
h = torch.empty(n, arch.d, device="cuda")
ws = m.workspace(1, n)
m.ci_forward_h(x.view(n, 3, 32, 32), h, ws)
xr = torch.empty(n, 3, 32, 32, device="cuda")
m.ci_inverse_h(h, xr, ws)
torch.cuda.synchronize()
np.savez(sys.argv[1], h=h.cpu().numpy(), xr=xr.cpu().numpy())
"""


@pytest.mark.parametrize("n", [5, 301, 1187])
def test_ts2_cluster_multicast_bit_exact(ci, tmp_path, n):
    """The cluster-multicast weight stream of k_stage_ts2 (CI_TS2_MC, read once per process: run in
    a subprocess) changes only where the weights come from and which CTA takes which batch: h and
    h^-1 are bit-identical to the default kernel, including the tails where one CTA of a pair has
    no batch (n = 5: 3 batches for one cluster; 1187: a partial last iteration)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mc in (False, True):
        env = dict(os.environ)
        env.pop("CI_TS2_MC", None)
        if mc:
            env["CI_TS2_MC"] = "1"
        f = str(tmp_path / f"mc{int(mc)}.npz")
        subprocess.run([sys.executable, "-c", _MC_SCRIPT, f, "fp32", str(n)], cwd=root, env=env, check=True,
                       timeout=300)
        out[mc] = np.load(f)
    assert np.array_equal(out[False]["h"], out[True]["h"])
    assert np.array_equal(out[False]["xr"], out[True]["xr"])
