"""ctypes front end of the f64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2106_06445_b200) never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 the oracle into oracle/liboracle.so (plain C, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-fno-fast-math",
                               "-ffp-contract=off", _SRC, "-o", _LIB + ".tmp", "-lpthread", "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class OrArch(ctypes.Structure):
    _fields_ = [("in_c", ctypes.c_int), ("in_h", ctypes.c_int), ("in_w", ctypes.c_int),
                ("n_stages", ctypes.c_int), ("squeeze", ctypes.c_int * 4),
                ("n_blocks", ctypes.c_int * 4), ("mid", ctypes.c_int * 4),
                ("act", ctypes.c_int), ("first_orient", ctypes.c_int),
                ("n_heads", ctypes.c_int), ("head_classes", ctypes.c_int * 4),
                ("enc_c1", ctypes.c_int), ("enc_mid", ctypes.c_int),
                ("block_kind", ctypes.c_int), ("fp_iters", ctypes.c_int)]


def to_orarch(arch) -> OrArch:
    a = OrArch()
    a.in_c, a.in_h, a.in_w = arch.in_c, arch.in_h, arch.in_w
    a.n_stages = len(arch.stages)
    for i, st in enumerate(arch.stages):
        a.squeeze[i], a.n_blocks[i], a.mid[i] = st.squeeze_before, st.n_blocks, st.mid
    a.act = arch.act_id
    a.first_orient = arch.first_orient
    a.n_heads = len(arch.heads)
    for i, c in enumerate(arch.heads):
        a.head_classes[i] = c
    if arch.encoder:
        a.enc_c1, a.enc_mid = arch.encoder
    a.block_kind = arch.block_id
    a.fp_iters = 0            # residual inverse: iterate to the 1e-12 step tolerance
    return a


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_d.restype = ctypes.c_long
        L.oracle_d.argtypes = [P]
        L.oracle_psi.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.oracle_psi_inv.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.oracle_conv3x3.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P]
        L.oracle_forward_h.argtypes = [P, P, ctypes.c_long, P, P, ctypes.c_int]
        L.oracle_inverse_h.argtypes = [P, P, ctypes.c_long, P, P, ctypes.c_int]
        L.oracle_mean.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_long, P, P]
        L.oracle_decode.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_long, P, P, P, P]
        L.oracle_classify.argtypes = [P, P, ctypes.c_int, ctypes.c_long, P, P, P]
        L.oracle_serve_group.argtypes = [P, P, ctypes.c_int, ctypes.c_long, P, P] + [P] * 9 + [ctypes.c_int, ctypes.c_int]
        L.oracle_encode_learned.argtypes = [P, P, ctypes.c_int, ctypes.c_long, P, P, ctypes.c_int]
        L.oracle_residual_inverse_block.restype = ctypes.c_int
        L.oracle_residual_inverse_block.argtypes = [P, P] + [ctypes.c_int] * 4 + [P, P, ctypes.c_int, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def default_threads() -> int:
    return os.cpu_count() or 1


# ---------------- primitives (exposed for pins) ----------------
def psi(x):
    x = _f64(x)
    C, H, W = x.shape
    out = np.empty((4 * C, H // 2, W // 2))
    lib().oracle_psi(_p(x), C, H, W, _p(out))
    return out


def psi_inv(x):
    x = _f64(x)
    C4, Ho, Wo = x.shape
    out = np.empty((C4 // 4, Ho * 2, Wo * 2))
    lib().oracle_psi_inv(_p(x), C4, Ho, Wo, _p(out))
    return out


def conv3x3(x, W, b):
    x, W, b = _f64(x), _f32(W), _f32(b)
    Cin, H, Wd = x.shape
    Cout = W.shape[0]
    out = np.empty((Cout, H, Wd))
    lib().oracle_conv3x3(_p(x), Cin, H, Wd, _p(W), _p(b), Cout, _p(out))
    return out


# ---------------- the hot-path operations ----------------
def forward_h(arch, params, x, nthreads=None):
    """x [n, C, H, W] -> h [n, d] (f64)."""
    x = _f64(x)
    n = x.shape[0]
    a, p = to_orarch(arch), _f32(params)
    out = np.empty((n, arch.d))
    lib().oracle_forward_h(ctypes.byref(a), _p(p), n, _p(x), _p(out), nthreads or default_threads())
    return out


def inverse_h(arch, params, h, nthreads=None, fp_iters=0):
    """h [n, d] -> x [n, C, H, W] (f64).  Residual archs: fp_iters fixed-point updates per
    block (0 = until the step is <= 1e-12, max 200)."""
    h = _f64(h)
    n = h.shape[0]
    a, p = to_orarch(arch), _f32(params)
    a.fp_iters = fp_iters
    out = np.empty((n, arch.in_c, arch.in_h, arch.in_w))
    lib().oracle_inverse_h(ctypes.byref(a), _p(p), n, _p(h), _p(out), nthreads or default_threads())
    return out


def mean(H):
    """H [B, k, d] -> m [B, d] = (sum_i H[b,i]) / k."""
    H = _f64(H)
    B, k, d = H.shape
    out = np.empty((B, d))
    lib().oracle_mean(k, B, d, _p(H), _p(out))
    return out


def decode(H, P, drop):
    """R = H with slot drop[b] replaced by k P[b] - sum_{i != drop[b]} H[b, i]."""
    H, P = _f64(H), _f64(P)
    drop = np.ascontiguousarray(drop, dtype=np.int32)
    B, k, d = H.shape
    out = np.empty_like(H)
    lib().oracle_decode(k, B, d, _p(H), _p(P), _p(drop), _p(out))
    return out


def classify(arch, params, head, z):
    z = _f64(z)
    n = z.shape[0]
    C = arch.heads[head]
    logits = np.empty((n, C))
    labels = np.empty(n, np.int32)
    a, p = to_orarch(arch), _f32(params)
    lib().oracle_classify(ctypes.byref(a), _p(p), head, n, _p(z), _p(logits), _p(labels))
    return logits, labels


def encode_perturbed(arch, params, H, eps, nthreads=None, fp_iters=0):
    """Perturbed exact encode: m = mean_i H_i + eps,
    x_p = h^-1(m).  H [B, k, d], eps [B, d] -> (m, x_p)."""
    m = mean(H) + _f64(eps)
    return m, inverse_h(arch, params, m, nthreads, fp_iters=fp_iters)


def residual_inverse_block(arch, params, stage, block, y, iters=0):
    """Fixed-point inverse of one residual block (stage, block) on y [C, H, W]:
    returns (x, number of updates)."""
    y = _f64(y)
    C, H, W = y.shape
    m = arch.stages[stage].mid
    a, p = to_orarch(arch), _f32(params)
    off = 0
    for s, (_, _, _, c, mm, nb) in enumerate(arch.stage_shapes()):
        per = mm * c * 9 + mm + c * mm * 9 + c
        if s == stage:
            off += block * per
            break
        off += nb * per
    x = np.empty_like(y)
    tmp = np.empty_like(y)
    hid = np.empty((m, H, W))
    it = lib().oracle_residual_inverse_block(ctypes.byref(a), _p(p[off:]), C, m, H, W, _p(y), _p(x), iters,
                                             _p(tmp), _p(hid))
    return x, it


def encode_learned(arch, params, x, nthreads=None):
    """Learned encoder (Arch E): x [B, k, C, H, W] -> x_p [B, C, H, W] (f64)."""
    x = _f64(x)
    B, k = x.shape[:2]
    a, p = to_orarch(arch), _f32(params)
    out = np.empty((B, arch.in_c, arch.in_h, arch.in_w))
    lib().oracle_encode_learned(ctypes.byref(a), _p(p), k, B, _p(x), _p(out), nthreads or default_threads())
    return out


def serve_group(arch, params, x, drop, nthreads=None, learned=False, fp_iters=0):
    """Whole coded path (exact encode, or the learned encoder when learned=True).
    x [B, k, C, H, W] fp32, drop [B] int32.

    Returns dict of f64 arrays: H, m, xp, P, R, logits[t], labels[t],
    logits_n[t], labels_n[t]  (t over heads)."""
    x = _f32(x)
    drop = np.ascontiguousarray(drop, dtype=np.int32)
    B, k = x.shape[:2]
    d = arch.d
    n = B * k
    a, p = to_orarch(arch), _f32(params)
    a.fp_iters = fp_iters
    H = np.empty((B, k, d)); m = np.empty((B, d))
    xp = np.empty((B, arch.in_c, arch.in_h, arch.in_w)); P = np.empty((B, d)); R = np.empty((B, k, d))
    ncls = sum(arch.heads)
    logits = np.empty(max(n * ncls, 1)); logits_n = np.empty(max(n * ncls, 1))
    labels = np.empty(max(n * len(arch.heads), 1), np.int32)
    labels_n = np.empty(max(n * len(arch.heads), 1), np.int32)
    lib().oracle_serve_group(ctypes.byref(a), _p(p), k, B, _p(x), _p(drop), _p(H), _p(m), _p(xp), _p(P),
                             _p(R), _p(logits), _p(labels), _p(logits_n), _p(labels_n),
                             nthreads or default_threads(), 1 if learned else 0)
    out = dict(H=H, m=m, xp=xp, P=P, R=R, logits=[], labels=[], logits_n=[], labels_n=[])
    lo = 0
    for t, C in enumerate(arch.heads):
        out["logits"].append(logits[lo:lo + n * C].reshape(B, k, C))
        out["logits_n"].append(logits_n[lo:lo + n * C].reshape(B, k, C))
        out["labels"].append(labels[t * n:(t + 1) * n].reshape(B, k))
        out["labels_n"].append(labels_n[t * n:(t + 1) * n].reshape(B, k))
        lo += n * C
    return out
