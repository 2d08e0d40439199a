"""Pins of the f64 CPU oracle against what the paper and the mathematics fix.

Each test names the pin id of SURVEY.md §8c and the passage it follows.  None
of these re-types the oracle's own formula: they compare against a library
routine (torch f64 conv2d / pixel_unshuffle), a closed form printed in the
paper, an invariant (volume preservation, linearity, round trip) or brute force.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import fixtures as fx
import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# ---------------------------------------------------------------- P6: library routines
def test_psi_is_pixel_unshuffle():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6, 8, 10))
    ref = Fnn.pixel_unshuffle(torch.from_numpy(x)[None], 2)[0].numpy()
    assert np.array_equal(oracle.psi(x), ref)
    assert np.array_equal(oracle.psi_inv(ref), x)
    ref_inv = Fnn.pixel_shuffle(torch.from_numpy(ref)[None], 2)[0].numpy()
    assert np.array_equal(oracle.psi_inv(ref), ref_inv)


@pytest.mark.parametrize("cin,cout,h,w", [(6, 64, 16, 16), (24, 7, 8, 8), (1, 3, 1, 1), (5, 4, 3, 7)])
def test_conv3x3_is_torch_conv2d_padding1(cin, cout, h, w):
    rng = np.random.default_rng(cin * 100 + cout)
    x = rng.standard_normal((cin, h, w))
    W = rng.standard_normal((cout, cin, 3, 3)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    ref = Fnn.conv2d(torch.from_numpy(x)[None], torch.from_numpy(W.astype(np.float64)),
                     torch.from_numpy(b.astype(np.float64)), padding=1)[0].numpy()
    assert rel(oracle.conv3x3(x, W, b), ref) < 1e-14


def torch_h(arch, params, x):
    """Independent f64 composition of h from torch library ops (pins block order,
    orientation, psi placement and the canonical parameter layout)."""
    p = {k: torch.from_numpy(v.astype(np.float64)) for k, v in fx.split_params(arch, params).items()}
    s = torch.from_numpy(np.asarray(x, np.float64))
    for si, (C, H, W, c, m, nb) in enumerate(arch.stage_shapes()):
        if arch.stages[si].squeeze_before:
            s = Fnn.pixel_unshuffle(s, 2)
        if arch.block == "residual":   # i-ResNet: s + G(s), G = conv -> ELU -> conv
            for t in range(nb):
                hid = Fnn.elu(Fnn.conv2d(s, p[f"s{si}b{t}.W1"], p[f"s{si}b{t}.b1"], padding=1))
                s = s + Fnn.conv2d(hid, p[f"s{si}b{t}.W2"], p[f"s{si}b{t}.b2"], padding=1)
            continue
        for t in range(nb):
            sa, sb = s[:, :c], s[:, c:]
            src, dst = (sa, sb) if ((arch.first_orient + t) & 1) == 0 else (sb, sa)
            hid = Fnn.conv2d(src, p[f"s{si}b{t}.W1"], p[f"s{si}b{t}.b1"], padding=1)
            if arch.act == "relu":
                hid = torch.relu(hid)
            upd = dst + Fnn.conv2d(hid, p[f"s{si}b{t}.W2"], p[f"s{si}b{t}.b2"], padding=1)
            s = torch.cat([sa, upd], 1) if ((arch.first_orient + t) & 1) == 0 else torch.cat([upd, sb], 1)
    return s.reshape(s.shape[0], -1).numpy()


@pytest.mark.parametrize("name", ["T", "M"])
def test_h_matches_torch_composition(name):
    arch = fx.ARCHS[name]
    params = fx.make_weights(arch, 5)
    x = fx.make_inputs(arch, 3, 1, 9)[:, 0]
    assert rel(oracle.forward_h(arch, params, x), torch_h(arch, params, x)) < 1e-12


def test_h_arch_c_one_image_matches_torch_composition():
    arch = fx.ARCH_C
    params = fx.make_weights(arch, 13)
    x = fx.make_inputs(arch, 1, 1, 3)[:, 0]
    assert rel(oracle.forward_h(arch, params, x), torch_h(arch, params, x)) < 1e-12


# ---------------------------------------------------------------- P1: linear worked example
def test_linear_worked_example_k2(golden):
    """PAPER.md:74-120 / 135: with linear f, Enc = f^-1((f(x1)+f(x2))/2) = (x1+x2)/2 and
    f(x2) is recovered from rows {1,3} as 2 r3 - r1 (Fig. 1 caption)."""
    g = golden("paper_eq1_worked_example.txt")
    Ginv = np.array(g["subset_inverse"], float).reshape(2, 2)
    arch = fx.linear_variant(fx.ARCH_T)
    params = fx.make_weights(arch, 11, zero_bias=True)
    x = fx.make_inputs(arch, 4, 2, 1)
    drop = np.ones(4, np.int32)  # worker 2 lost
    out = oracle.serve_group(arch, params, x, drop)
    # encoded query is the plain average (linearity)
    assert rel(out["xp"], x.astype(np.float64).mean(1)) < 1e-12
    # f((x1+x2)/2) = (f(x1)+f(x2))/2
    assert rel(out["P"], out["H"].mean(1)) < 1e-12
    # decode via the paper's printed subset inverse applied to [r1; r3]
    r1, r3 = out["H"][:, 0], out["P"]
    f2 = Ginv[1, 0] * r1 + Ginv[1, 1] * r3
    assert rel(out["R"][:, 1], f2) < 1e-13
    assert rel(out["R"][:, 1], out["H"][:, 1]) < 1e-12
    # any two rows of G are invertible
    G = np.array(g["G"], float).reshape(3, 2)
    for i in range(3):
        for j in range(i + 1, 3):
            assert abs(np.linalg.det(G[[i, j]])) > 0.25


def test_linear_h_jacobian_volume_preserving():
    """P6: Arch T, identity act, zero bias => h(x) = J x with |det J| = 1 (additive coupling
    has unit Jacobian determinant, psi is a permutation)."""
    arch = fx.linear_variant(fx.ARCH_T)
    params = fx.make_weights(arch, 3, zero_bias=True)
    d = arch.d
    E = np.eye(d).reshape(d, arch.in_c, arch.in_h, arch.in_w)
    J = oracle.forward_h(arch, params, E).T          # column i = h(e_i)
    x = fx.make_inputs(arch, 2, 1, 4)[:, 0].astype(np.float64)
    assert rel(oracle.forward_h(arch, params, x), (J @ x.reshape(2, -1).T).T) < 1e-12
    sign, logdet = np.linalg.slogdet(J)
    assert abs(logdet) < 1e-10


def test_nonlinearity_witness():
    """with ReLU, h((x1+x2)/2) != (h(x1)+h(x2))/2 by > 1e-3."""
    arch = fx.ARCH_T
    params = fx.make_weights(arch, 11)
    x = fx.make_inputs(arch, 1, 2, 1)[0].astype(np.float64)
    hx = oracle.forward_h(arch, params, x)
    hm = oracle.forward_h(arch, params, x.mean(0, keepdims=True))
    assert np.max(np.abs(hm[0] - hx.mean(0))) > 1e-3


# ---------------------------------------------------------------- P2: rotation (App. A.1)
def test_rotation_as_three_shears(golden):
    g = golden("rotation_app_a1.txt")
    theta = float(g["theta"][0])
    assert abs(theta - math.pi / 3) < 1e-16
    params = fx.rotation_params(theta)
    e1 = np.array([1.0, 0.0]).reshape(1, 2, 1, 1)
    y = oracle.forward_h(fx.ARCH_R, params, e1)[0]
    # parameters are fp32 by design (fixtures), so the shear coefficients carry fp32
    # rounding (|delta| <= 2^-24 relative): the rotation is reproduced to ~1e-7.
    assert np.max(np.abs(y - np.array(g["f_of_e1"], float))) < 1e-7
    # the full rotation matrix and its inverse
    E = np.eye(2).reshape(2, 2, 1, 1)
    Rm = oracle.forward_h(fx.ARCH_R, params, E).T
    Rref = np.array([[math.cos(theta), -math.sin(theta)], [math.sin(theta), math.cos(theta)]])
    assert np.max(np.abs(Rm - Rref)) < 1e-7
    Rinv = oracle.inverse_h(fx.ARCH_R, params, np.eye(2)).reshape(2, 2).T
    assert np.max(np.abs(Rinv - Rref.T)) < 1e-7
    assert np.max(np.abs(Rinv @ Rm - np.eye(2))) < 1e-15   # exact inverse of the fp32 map


def test_app_a1_reconstruction_error_band(golden):
    """PAPER.md:788-797 with reading Q12: parity input = (sum_j x_j)/k over all j,
    f(x_a) recovered as k f(parity) - sum_{j!=a} f(x_j), then x_a = f^-1(.).
    Mean ||x_a - x^_a||_2 over trials must fall in the printed band (relaxed)."""
    g = golden("rotation_app_a1.txt")
    theta = float(g["theta"][0])
    lo, hi = (float(v) for v in g["error_band"])
    mu = np.array(g["mixture_means"], float).reshape(2, 2)
    params = fx.rotation_params(theta)
    rng = np.random.default_rng(2106)
    trials = 2000
    for k in (int(v) for v in g["k_values"]):
        comp = rng.integers(0, 2, size=(trials, k))
        xs = mu[comp] + rng.standard_normal((trials, k, 2))
        a = rng.integers(0, k, size=trials)
        fx_all = oracle.forward_h(fx.ARCH_R, params, xs.reshape(-1, 2, 1, 1)).reshape(trials, k, 2)
        xbar = xs.mean(1)
        fpar = oracle.forward_h(fx.ARCH_R, params, xbar.reshape(-1, 2, 1, 1))
        mask = np.ones((trials, k), bool)
        mask[np.arange(trials), a] = False
        fa_hat = k * fpar - (fx_all * mask[..., None]).sum(1)
        xa_hat = oracle.inverse_h(fx.ARCH_R, params, fa_hat).reshape(trials, 2)
        err = np.linalg.norm(xs[np.arange(trials), a] - xa_hat, axis=1).mean()
        assert lo <= err <= hi, (k, err)


# ---------------------------------------------------------------- P3/P4/P5: exactness
@pytest.mark.parametrize("name,n", [("T", 4), ("M", 3), ("C", 1)])
def test_round_trip(name, n):
    """P3: h^-1(h(x)) = x and h(h^-1(y)) = y."""
    arch = fx.ARCHS[name]
    params = fx.make_weights(arch, 21)
    x = fx.make_inputs(arch, n, 1, 22)[:, 0].astype(np.float64)
    h = oracle.forward_h(arch, params, x)
    assert rel(oracle.inverse_h(arch, params, h), x) < 1e-13
    y = h[::-1].copy()
    assert rel(oracle.forward_h(arch, params, oracle.inverse_h(arch, params, y)), y) < 1e-13


@pytest.mark.parametrize("cfg", ["C1", "C2small"])
def test_exact_recovery_and_input_recovery(cfg):
    """P4: with the ideal encoder the decoded features equal the
    lost worker's h(x_j); P5: h^-1 of them returns x_j."""
    if cfg == "C1":
        c = fx.CONFIGS["C1"]
        arch, k, B = c.arch, c.k, c.B
        params, x, drop = fx.make_weights(arch, c.seed_w), fx.make_inputs(arch, B, k, c.seed_x), \
            fx.make_drops(B, k, c.seed_drop)
    else:
        arch, k, B = fx.ARCH_M, 4, 6
        params, x, drop = fx.make_weights(arch, 12), fx.make_inputs(arch, B, k, 2), fx.make_drops(B, k, 102)
    out = oracle.serve_group(arch, params, x, drop)
    bi = np.arange(B)
    assert rel(out["R"][bi, drop], out["H"][bi, drop]) < 1e-12
    xr = oracle.inverse_h(arch, params, out["R"][bi, drop])
    assert rel(xr, x[bi, drop]) < 1e-12
    # labels of the decoded slot equal the normal labels
    for t in range(len(arch.heads)):
        assert np.array_equal(out["labels"][t], out["labels_n"][t])


# ---------------------------------------------------------------- P10: amplification law
def test_amplification_law():
    """PAPER.md:299-306 (SURVEY Q10 reading): if f(x_{k+1}) = mean + eps then
    f^(x_a) - f(x_a) = k eps."""
    rng = np.random.default_rng(7)
    for k in (2, 4, 10):
        B, d = 5, 17
        H = rng.standard_normal((B, k, d))
        eps = 1e-3 * rng.standard_normal((B, d))
        P = oracle.mean(H) + eps
        drop = rng.integers(0, k, B).astype(np.int32)
        R = oracle.decode(H, P, drop)
        err = R[np.arange(B), drop] - H[np.arange(B), drop]
        assert np.max(np.abs(err - k * eps)) < 1e-12


# ---------------------------------------------------------------- P11-style exact integer checks
def test_mean_and_decode_integer_exact():
    rng = np.random.default_rng(3)
    for k in (1, 2, 3, 4, 10):
        B, d = 7, 33
        H = rng.integers(-1024, 1024, size=(B, k, d)).astype(np.float64) * k
        m = oracle.mean(H)
        assert np.array_equal(m, H.sum(1) / k)
        drop = rng.integers(-1, k, B).astype(np.int32)
        R = oracle.decode(H, m, drop)
        assert np.array_equal(R, H)  # exact mean as parity => exact recovery


# ---------------------------------------------------------------- P16: degenerate cases
def test_degenerate_k1_and_no_drop():
    arch = fx.ARCH_T
    params = fx.make_weights(arch, 11)
    x = fx.make_inputs(arch, 3, 1, 1)
    out = oracle.serve_group(arch, params, x, np.zeros(3, np.int32))
    assert rel(out["xp"], x[:, 0]) < 1e-12            # repetition code: x_p = x_1
    assert np.array_equal(out["R"][:, 0], out["P"])     # decode = 1 * P
    x2 = fx.make_inputs(arch, 2, 2, 1)
    out2 = oracle.serve_group(arch, params, x2, np.full(2, -1, np.int32))
    assert np.array_equal(out2["R"], out2["H"])         # no loss: untouched


# ---------------------------------------------------------------- P12: argmax ties
def test_classify_lowest_index_tie_and_brute_force():
    arch = fx.ARCH_T
    params = fx.make_weights(arch, 11).copy()
    p = fx.split_params(arch, params)
    z = np.random.default_rng(1).standard_normal((6, arch.d))
    logits, labels = oracle.classify(arch, params, 0, z)
    W, b = p["g0.W"].astype(np.float64), p["g0.b"].astype(np.float64)
    assert rel(logits, z @ W.T + b) < 1e-13   # brute force matrix product
    assert np.array_equal(labels, np.argmax(logits, 1))
    # construct exact ties: rows 3 and 7 of W identical, bias equal, and dominant
    p["g0.W"][7] = p["g0.W"][3]
    p["g0.b"][7] = p["g0.b"][3] = 10.0
    logits, labels = oracle.classify(arch, params, 0, z)
    assert np.all(logits[:, 3] == logits[:, 7]) and np.all(labels == 3)


# ---------------------------------------------------------------- a0: group assignment / drops
def test_splitmix64_reference_vectors(golden):
    g = golden("splitmix64.txt")
    got = fx.splitmix64_at(1234567, np.arange(5))
    assert [int(v) for v in got] == [int(v) for v in g["seed_1234567"]]
    got0 = fx.splitmix64_at(0, np.arange(3))
    assert [int(v) for v in got0] == [int(v, 16) for v in g["seed_0_hex"]]


def test_group_assignment_and_drops():
    q = np.arange(1000)
    b, i = fx.group_of(q, 7)
    assert np.array_equal(b * 7 + i, q) and i.max() == 6
    drops = fx.make_drops(100000, 10, 103)
    assert drops.min() == 0 and drops.max() == 9
    counts = np.bincount(drops, minlength=10)
    assert np.all(np.abs(counts - 10000) < 500)   # uniform one-of-k
    # counter-based: element b depends only on (seed, b)
    assert np.array_equal(fx.make_drops(50, 10, 103), drops[:50])


# ---------------------------------------------------------------- learned encoder (a3', C4)
def torch_encoder(arch, params, x):
    """Independent f64 composition of Arch E from torch library ops."""
    p = {k: torch.from_numpy(v.astype(np.float64)) for k, v in fx.split_params(arch, params).items()}
    xt = torch.from_numpy(np.asarray(x, np.float64))           # [B, k, C, H, W]
    B, k = xt.shape[:2]
    e = torch.relu(Fnn.conv2d(xt.reshape(B * k, *xt.shape[2:]), p["E1.W"], p["E1.b"], padding=1))
    m = e.reshape(B, k, *e.shape[1:]).mean(1)
    z = Fnn.pixel_unshuffle(m, 2)
    z = torch.relu(Fnn.conv2d(z, p["E2.W"], p["E2.b"], padding=1))
    z = torch.relu(Fnn.conv2d(z, p["E3.W"], p["E3.b"], padding=1))
    u = Fnn.pixel_shuffle(z, 2) + m
    return Fnn.conv2d(u, p["E4.W"], p["E4.b"], padding=1).numpy()


@pytest.mark.parametrize("name,k", [("TE", 3), ("CE", 2)])
def test_learned_encoder_matches_torch_composition(name, k):
    arch = fx.ARCHS[name]
    params = fx.make_weights(arch, 14)
    x = fx.make_inputs(arch, 2, k, 4)
    assert rel(oracle.encode_learned(arch, params, x), torch_encoder(arch, params, x)) < 1e-12


def test_learned_encoder_permutation_and_copy_invariance():
    """P14 (PAPER.md:411 'permutation invariance ... average after the first layer'):
    permuting the k inputs leaves x_p unchanged; k copies of one image encode like k = 1."""
    arch = fx.ARCH_TE
    params = fx.make_weights(arch, 14)
    x = fx.make_inputs(arch, 3, 5, 4)
    xp = oracle.encode_learned(arch, params, x)
    perm = np.array([3, 0, 4, 1, 2])
    assert rel(oracle.encode_learned(arch, params, x[:, perm]), xp) < 1e-14
    one = x[:, :1]
    assert rel(oracle.encode_learned(arch, params, np.repeat(one, 4, axis=1)),
               oracle.encode_learned(arch, params, one)) < 1e-14


def test_serve_group_learned_decode_algebra():
    """With the learned encoder the parity is only approximate, but the decode algebra still
    gives f^(x_j) = k P - sum_{i != j} H_i exactly."""
    arch = fx.ARCH_TE
    params = fx.make_weights(arch, 14)
    x = fx.make_inputs(arch, 4, 3, 4)
    drop = fx.make_drops(4, 3, 104)
    out = oracle.serve_group(arch, params, x, drop, learned=True)
    assert rel(out["xp"], oracle.encode_learned(arch, params, x)) < 1e-15
    assert rel(out["P"], oracle.forward_h(arch, params, out["xp"])) < 1e-15
    bi = np.arange(4)
    H = out["H"]
    mask = np.ones((4, 3), bool); mask[bi, drop] = False
    ref = 3 * out["P"] - (H * mask[..., None]).sum(1)
    assert rel(out["R"][bi, drop], ref) < 1e-13
    assert len(out["logits"]) == 2 and out["logits"][1].shape == (4, 3, 2)


# ---------------------------------------------------------------- P7: i-ResNet variant (f1)
ARCH_P7 = fx.Arch("P7", 1, 1, 1, (fx.Stage(0, 1, 1),), act="elu", block="residual", heads=())


def p7_params():
    """G(x) = 0.5 * ELU(x + 10) - 5 = 0.5 x for x > -10: on a 1x1 image only the
    centre taps act; the off-centre taps are junk that zero padding must ignore."""
    w1 = np.full((1, 1, 3, 3), 7.0, np.float32); w1[0, 0, 1, 1] = 1.0
    w2 = np.full((1, 1, 3, 3), -3.0, np.float32); w2[0, 0, 1, 1] = 0.5
    return np.concatenate([w1.ravel(), [10.0], w2.ravel(), [-5.0]]).astype(np.float32)


def test_fixed_point_closed_form_rate_half():
    """f(x) = 1.5 x: h(2) = 3; N updates of x <- 3 - 0.5 x from x_0 = 3 give exactly
    2 + (-1/2)^N (dyadic, exact in f64); the converged inverse meets the 1e-12 step rule within
    ceil(log(tol / |x_0 - x*|) / log L) + 2 updates."""
    params = p7_params()
    x = np.array([[[[2.0]]]])
    assert oracle.forward_h(ARCH_P7, params, x)[0, 0] == 3.0
    for N in (1, 2, 5, 10, 30):
        xi, it = oracle.residual_inverse_block(ARCH_P7, params, 0, 0, np.array([[[3.0]]]), iters=N)
        assert it == N and xi[0, 0, 0] == 2.0 + (-0.5) ** N
        assert oracle.inverse_h(ARCH_P7, params, np.array([[3.0]]), fp_iters=N)[0, 0, 0, 0] == 2.0 + (-0.5) ** N
    xi, it = oracle.residual_inverse_block(ARCH_P7, params, 0, 0, np.array([[[3.0]]]))
    assert abs(xi[0, 0, 0] - 2.0) <= 1e-12 and it <= math.ceil(math.log(1e-12) / math.log(0.5)) + 2


def test_spectral_norm_matches_svd_of_conv_operator():
    """The fixtures' power iteration (weight prep) against the largest singular
    value of the explicit zero-padded conv matrix (numpy SVD)."""
    rng = np.random.default_rng(3)
    for ci, co, H, W in ((12, 16, 4, 4), (5, 7, 3, 5)):
        w = rng.standard_normal((co, ci, 3, 3))
        A = np.zeros((co * H * W, ci * H * W))
        for j in range(ci * H * W):
            e = np.zeros(ci * H * W); e[j] = 1.0
            A[:, j] = fx._conv_nobias(e.reshape(ci, H, W), w).ravel()
        smax = np.linalg.svd(A, compute_uv=False)[0]
        # power iteration approaches sigma_max from below (Rayleigh quotient of A^T A)
        for iters, tol in ((200, 1e-6), (60, 2e-2)):
            est = fx.conv_spectral_norm(w, H, W, iters=iters)
            assert smax * (1 - tol) <= est <= smax * (1 + 1e-12), (iters, est, smax)
        # the adjoint really is the transpose
        y = rng.standard_normal((co, H, W))
        assert np.allclose(fx._conv_adjoint(y, w).ravel(), A.T @ y.ravel(), atol=1e-12)


def test_residual_h_matches_torch_composition():
    arch = fx.ARCH_TR
    params = fx.make_weights(arch, 5)
    x = fx.make_inputs(arch, 3, 1, 9)[:, 0]
    assert rel(oracle.forward_h(arch, params, x), torch_h(arch, params, x)) < 1e-12


def test_residual_arch_c_one_image_matches_torch_composition():
    arch = fx.ARCH_CR
    params = fx.make_weights(arch, 13)
    x = fx.make_inputs(arch, 1, 1, 3)[:, 0]
    assert rel(oracle.forward_h(arch, params, x), torch_h(arch, params, x)) < 1e-12


def test_residual_blocks_are_contractions():
    """Lip(G) <= L = 0.9 for every block of Arch TR (spectral normalisation + 1-Lipschitz ELU):
    random pairs, ||G(u) - G(v)||_2 <= L ||u - v||_2 (G from the oracle's own block: y - x)."""
    arch = fx.ARCH_TR
    params = fx.make_weights(arch, 5)
    one = fx.Arch("TR1", 12, 4, 4, (fx.Stage(0, 1, 16),), act="elu", block="residual", heads=())
    per = fx.n_params(one)
    rng = np.random.default_rng(0)
    for t in range(2):
        blk = params[t * per:(t + 1) * per]
        for _ in range(20):
            u = rng.standard_normal((2, 12, 4, 4)) * rng.uniform(0.01, 3)
            v = u + rng.standard_normal((2, 12, 4, 4)) * rng.uniform(1e-3, 1)
            gu = oracle.forward_h(one, blk, u) - u.reshape(2, -1)
            gv = oracle.forward_h(one, blk, v) - v.reshape(2, -1)
            for i in range(2):
                assert np.linalg.norm(gu[i] - gv[i]) <= arch.lip * np.linalg.norm((u - v)[i]) * (1 + 1e-9)


def test_residual_round_trip_and_iteration_bound():
    """h^-1(h(x)) = x for the converged fixed point; per-block update counts respect the
    geometric bound ceil(log(tol / ||x_0 - x*||_inf) / log L) + 2."""
    arch = fx.ARCH_TR
    params = fx.make_weights(arch, 5)
    x = fx.make_inputs(arch, 4, 1, 2)[:, 0]
    h = oracle.forward_h(arch, params, x)
    assert np.abs(oracle.inverse_h(arch, params, h) - x).max() < 1e-11
    # block 1 of the only stage: y = h (as a state), x* = state before block 1
    one = fx.Arch("TR1", 12, 4, 4, (fx.Stage(0, 1, 16),), act="elu", block="residual", heads=())
    per = fx.n_params(one)
    s0 = oracle.psi(x[0])                                   # state entering block 0
    s1 = oracle.forward_h(one, params[:per], s0[None])[0].reshape(s0.shape)
    y = oracle.forward_h(one, params[per:2 * per], s1[None])[0].reshape(s0.shape)
    xs, it = oracle.residual_inverse_block(arch, params, 0, 1, y)
    assert np.abs(xs - s1).max() < 1e-11
    bound = math.ceil(math.log(1e-12 / np.abs(y - s1).max()) / math.log(arch.lip)) + 2
    assert it <= bound, (it, bound)
    # fixed N: error decays at least geometrically in N
    errs = [np.abs(oracle.residual_inverse_block(arch, params, 0, 1, y, iters=N)[0] - s1).max() for N in (2, 4, 8)]
    assert errs[0] > errs[1] > errs[2] and errs[2] <= arch.lip ** 8 * np.abs(y - s1).max()


# ---------------------------------------------------------------- f4: perturbed encode
def test_perturbed_encode_zero_noise_and_k_eps_law():
    """sigma = 0 is the ideal encode bitwise; through an exactly invertible f,
    h(x_p) = mean + eps, so decoding the lost slot returns f(x_a) + k eps."""
    arch = fx.ARCH_T
    params = fx.make_weights(arch, 3)
    B, k = 6, 4
    x = fx.make_inputs(arch, B, k, 2)
    H = oracle.forward_h(arch, params, x.reshape(B * k, *x.shape[2:])).reshape(B, k, -1)
    m0, xp0 = oracle.encode_perturbed(arch, params, H, np.zeros((B, arch.d)))
    assert np.array_equal(xp0, oracle.inverse_h(arch, params, oracle.mean(H)))
    eps = 1e-2 * np.random.default_rng(1).standard_normal((B, arch.d))
    m, xp = oracle.encode_perturbed(arch, params, H, eps)
    P = oracle.forward_h(arch, params, xp)
    assert np.max(np.abs(P - (oracle.mean(H) + eps))) < 1e-12
    drop = np.arange(B, dtype=np.int32) % k
    R = oracle.decode(H, P, drop)
    err = R[np.arange(B), drop] - H[np.arange(B), drop]
    assert np.max(np.abs(err - k * eps)) < 1e-11
