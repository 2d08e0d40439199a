"""Thin ctypes binding of libcodedinv.so (include/codedinv.h).

Argument marshalling only: every step of the coded path runs in the library's CUDA
kernels.  Tensors are torch CUDA tensors (device memory / streams come from PyTorch);
the host-buffer entry point takes numpy arrays.  If the shared library is missing this
module raises at import time -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcodedinv.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

CI_OK, CI_ERR_INVALID_ARG, CI_ERR_INVALID_SHAPE, CI_ERR_DIM_MISMATCH, CI_ERR_UNSUPPORTED, \
    CI_ERR_WORKSPACE, CI_ERR_CUDA, CI_ERR_UNDECODABLE, CI_ERR_COMM = range(9)
CI_SHARD_GROUPS, CI_SHARD_WORKERS = 0, 1
CI_COMM_ID_BYTES = 128
CI_FIRSTK_CODED, CI_FIRSTK_UNCODED = 0, 1
CI_PREC_FP32, CI_PREC_BF16, CI_PREC_F16X2 = 0, 1, 2
CI_ENC_EXACT, CI_ENC_LEARNED = 0, 1
PRECISIONS = {"fp32": CI_PREC_FP32, "bf16": CI_PREC_BF16, "f16x2": CI_PREC_F16X2}

EXPORTS = ["ci_last_error", "ci_model_create", "ci_model_destroy", "ci_feature_dim",
           "ci_workspace_size", "ci_check", "ci_forward_h", "ci_inverse_h", "ci_encode",
           "ci_decode", "ci_classify", "ci_serve_group", "ci_workspace_size_host",
           "ci_serve_group_host", "ci_make_drops", "ci_comm_unique_id", "ci_comm_create", "ci_comm_destroy",
           "ci_workspace_size_general", "ci_encode_general", "ci_decode_general", "ci_serve_general",
           "ci_encode_perturbed", "ci_online_update", "ci_serve_group_host_async", "ci_workspace_size_first_k",
           "ci_serve_first_k"]
TESTING_EXPORTS = ["ci_test_prof_enable", "ci_test_prof_read", "ci_test_launch_count", "ci_test_mean",
                   "ci_test_plan", "ci_test_rendezvous"]  # include/codedinv_testing.h


class CiStage(ctypes.Structure):
    _fields_ = [("squeeze_before", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
                ("mid_channels", ctypes.c_int32)]


class CiArch(ctypes.Structure):
    _fields_ = [("in_c", ctypes.c_int32), ("in_h", ctypes.c_int32), ("in_w", ctypes.c_int32),
                ("n_stages", ctypes.c_int32), ("stage", CiStage * 4), ("act", ctypes.c_int32),
                ("first_orientation", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("head_classes", ctypes.c_int32 * 4), ("enc_c1", ctypes.c_int32), ("enc_mid", ctypes.c_int32),
                ("block_kind", ctypes.c_int32), ("fp_iters", ctypes.c_int32)]


_P, _I32, _I64, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_sig = {
    "ci_last_error": (ctypes.c_char_p, []),
    "ci_model_create": (_I32, [_P, _P, _SZ, _I32, ctypes.c_int, _P]),
    "ci_model_destroy": (None, [_P]),
    "ci_feature_dim": (_I64, [_P]),
    "ci_workspace_size": (_I32, [_P, _I32, _I64, _P]),
    "ci_check": (_I32, [_P, _P, _SZ, _P]),
    "ci_forward_h": (_I32, [_P, _P, _P, _I64, _P, _SZ, _P]),
    "ci_inverse_h": (_I32, [_P, _P, _P, _I64, _P, _SZ, _P]),
    "ci_encode": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_decode": (_I32, [_I32, _I64, _I64, _P, _P, _P, _P, _SZ, _P]),
    "ci_classify": (_I32, [_P, _I32, _P, _I64, _P, _P, _P]),
    "ci_serve_group": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_workspace_size_host": (_I32, [_P, _I32, _I64, _P]),
    "ci_serve_group_host": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_serve_group_host_async": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_make_drops": (_I32, [_I32, _I64, ctypes.c_uint64, _P, _P]),
    "ci_workspace_size_first_k": (_I32, [_P, _I32, _I32, _P]),
    "ci_serve_first_k": (_I32, [_P, _I32, _I32, _I64, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_comm_unique_id": (_I32, [_P]),
    "ci_comm_create": (_I32, [_P, _I32, _I32, _I32, _I64, _I64, ctypes.c_int, _P]),
    "ci_comm_destroy": (None, [_P]),
    "ci_test_rendezvous": (_I32, [_P, _I32, _I32, _P, _I32, _P]),
    "ci_workspace_size_general": (_I32, [_P, _I32, _I32, _I64, _P]),
    "ci_encode_perturbed": (_I32, [_P, _I32, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_online_update": (_I32, [_I32, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_encode_general": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_decode_general": (_I32, [_I32, _I32, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_serve_general": (_I32, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ci_test_prof_enable": (_I32, [_I32]),
    "ci_test_prof_read": (_I32, [_P, _P, _P]),
    "ci_test_launch_count": (_I64, [_I32]),
    "ci_test_mean": (_I32, [_I32, _I64, _I64, _P, _P, _P]),
    "ci_test_plan": (_I32, [_I32, _I32, _I32, _I32, _I32, _P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args


class CiError(RuntimeError):
    def __init__(self, status, where):
        super().__init__(f"{where}: status {status}: {_lib.ci_last_error().decode()}")
        self.status = status


def _check(status, where):
    if status != CI_OK:
        raise CiError(status, where)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def to_ci_arch(arch) -> CiArch:
    a = CiArch()
    a.in_c, a.in_h, a.in_w = arch.in_c, arch.in_h, arch.in_w
    a.n_stages = len(arch.stages)
    for i, st in enumerate(arch.stages):
        a.stage[i].squeeze_before, a.stage[i].n_blocks, a.stage[i].mid_channels = \
            st.squeeze_before, st.n_blocks, st.mid
    a.act = arch.act_id
    a.first_orientation = arch.first_orient
    a.n_heads = len(arch.heads)
    for i, c in enumerate(arch.heads):
        a.head_classes[i] = c
    if getattr(arch, "encoder", ()):
        a.enc_c1, a.enc_mid = arch.encoder
    a.block_kind = {"coupling": 0, "residual": 1}[getattr(arch, "block", "coupling")]
    a.fp_iters = getattr(arch, "fp_iters", 0) if a.block_kind else 0
    return a


class Model:
    """Owns a ci_model_t.  `params` is the canonical flat fp32 vector (numpy)."""

    def __init__(self, arch, params, precision="fp32", device=0):
        self.arch = arch
        self.precision = precision
        p = np.ascontiguousarray(params, dtype=np.float32)
        self._carch = to_ci_arch(arch)
        h = ctypes.c_void_p()
        _check(_lib.ci_model_create(ctypes.byref(self._carch), _ptr(p), p.size,
                                    PRECISIONS[precision], device, ctypes.byref(h)), "ci_model_create")
        self._h = h
        self.d = int(_lib.ci_feature_dim(h))

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:   # (module globals may be gone at exit)
            _lib.ci_model_destroy(self._h)
            self._h = None

    __del__ = close

    # ---- workspace
    def workspace_size(self, k, B):
        n = ctypes.c_size_t()
        _check(_lib.ci_workspace_size(self._h, k, B, ctypes.byref(n)), "ci_workspace_size")
        return n.value

    def workspace_size_host(self, k, B):
        n = ctypes.c_size_t()
        _check(_lib.ci_workspace_size_host(self._h, k, B, ctypes.byref(n)), "ci_workspace_size_host")
        return n.value

    def workspace(self, k, B, host=False):
        import torch
        n = self.workspace_size_host(k, B) if host else self.workspace_size(k, B)
        return torch.zeros(n, dtype=torch.uint8, device="cuda")

    def workspace_general(self, k, r, B):
        import torch
        n = ctypes.c_size_t()
        _check(_lib.ci_workspace_size_general(self._h, k, r, B, ctypes.byref(n)), "ci_workspace_size_general")
        return torch.zeros(n.value, dtype=torch.uint8, device="cuda")

    def ci_encode_perturbed(self, h, eps, x_parity, ws, mean_out=None, stream=None):
        B, k = h.shape[0], h.shape[1]
        _check(_lib.ci_encode_perturbed(self._h, k, B, _ptr(h), _ptr(eps), _ptr(x_parity), _ptr(mean_out),
                                        _ptr(ws), ws.numel(), _stream(stream)), "ci_encode_perturbed")

    # ---- general (n, k) codes: coef [r][k] device fp32, avail [B] device uint32 (as int32)
    def ci_encode_general(self, coef, h, x_parity, ws, comb_out=None, stream=None):
        r, k = coef.shape
        B = h.shape[0]
        _check(_lib.ci_encode_general(self._h, k, r, B, _ptr(coef), _ptr(h), _ptr(x_parity), _ptr(comb_out),
                                      _ptr(ws), ws.numel(), _stream(stream)), "ci_encode_general")

    def ci_serve_general(self, coef, x, avail, h_out, h_parity, ws, x_parity=None, logits=None, labels=None,
                         stream=None):
        r, k = coef.shape
        B = x.shape[0]
        _check(_lib.ci_serve_general(self._h, k, r, B, _ptr(coef), _ptr(x), _ptr(avail), _ptr(h_out),
                                     _ptr(h_parity), _ptr(x_parity), _ptr(logits), _ptr(labels), _ptr(ws),
                                     ws.numel(), _stream(stream)), "ci_serve_general")

    # ---- ABI calls (same names as the C entry points)
    def ci_forward_h(self, x, h, ws, stream=None):
        _check(_lib.ci_forward_h(self._h, _ptr(x), _ptr(h), x.shape[0], _ptr(ws), ws.numel(),
                                 _stream(stream)), "ci_forward_h")

    def ci_inverse_h(self, h, x, ws, stream=None):
        _check(_lib.ci_inverse_h(self._h, _ptr(h), _ptr(x), h.shape[0], _ptr(ws), ws.numel(),
                                 _stream(stream)), "ci_inverse_h")

    def ci_encode(self, h, x_parity, ws, mean_out=None, stream=None, x=None, learned=False):
        """Exact mode: h [B, k, d].  Learned mode (learned=True): x [B, k, C, H, W]."""
        src = x if learned else h
        B, k = src.shape[0], src.shape[1]
        _check(_lib.ci_encode(self._h, CI_ENC_LEARNED if learned else CI_ENC_EXACT, k, B, _ptr(x), _ptr(h),
                              _ptr(x_parity), _ptr(mean_out), _ptr(ws), ws.numel(), _stream(stream)), "ci_encode")

    def ci_classify(self, head, z, logits, labels=None, stream=None):
        _check(_lib.ci_classify(self._h, head, _ptr(z), z.shape[0], _ptr(logits), _ptr(labels),
                                _stream(stream)), "ci_classify")

    def ci_serve_group(self, x, drop, h_out, h_parity, ws, x_parity=None, logits=None, labels=None,
                       stream=None, learned=False, comm=None, k=None):
        """comm: a Comm (CI_SHARD_WORKERS: this rank's worker; x is its slot [B, C, H, W], or the
        parity rank's [B, k, C, H, W] / None, so k must be given)."""
        if comm is not None and comm.layout == CI_SHARD_WORKERS:
            B, k = drop.shape[0], comm.nranks - 1
        else:
            B, k = x.shape[0], x.shape[1]
        _check(_lib.ci_serve_group(self._h, CI_ENC_LEARNED if learned else CI_ENC_EXACT, k, B, _ptr(x), _ptr(drop),
                                   _ptr(h_out), _ptr(h_parity), _ptr(x_parity), _ptr(logits), _ptr(labels),
                                   comm._h if comm is not None else None, _ptr(ws), ws.numel(), _stream(stream)),
               "ci_serve_group")

    def ci_serve_group_host(self, x, drop, h_out, h_parity, logits, labels, ws, stream=None, learned=False,
                            sync=True):
        """sync=False: ci_serve_group_host_async (returns after enqueueing; sync the stream)."""
        B, k = x.shape[0], x.shape[1]
        fn = _lib.ci_serve_group_host if sync else _lib.ci_serve_group_host_async
        _check(fn(self._h, CI_ENC_LEARNED if learned else CI_ENC_EXACT, k, B, _ptr(x), _ptr(drop), _ptr(h_out),
                  _ptr(h_parity), _ptr(logits), _ptr(labels), _ptr(ws), ws.numel(), _stream(stream)),
               "ci_serve_group_host")

    def workspace_first_k(self, k, max_inflight):
        import torch
        n = ctypes.c_size_t()
        _check(_lib.ci_workspace_size_first_k(self._h, k, max_inflight, ctypes.byref(n)), "ci_workspace_size_first_k")
        return torch.zeros(n.value, dtype=torch.uint8, device="cuda")

    def ci_serve_first_k(self, x, straggler, delay_ns, features, logits, labels, records, ws, max_inflight=32,
                         uncoded=False, stream=None):
        """x [Q, k, C, H, W] device; straggler: numpy int32 [Q] (host); records int64 [Q, 4] device."""
        Q, k = x.shape[0], x.shape[1]
        st = np.ascontiguousarray(straggler, dtype=np.int32)
        _check(_lib.ci_serve_first_k(self._h, CI_FIRSTK_UNCODED if uncoded else CI_FIRSTK_CODED, k, Q, _ptr(x),
                                     _ptr(st), int(delay_ns), max_inflight, _ptr(features), _ptr(logits),
                                     _ptr(labels), _ptr(records), _ptr(ws), ws.numel(), _stream(stream)),
               "ci_serve_first_k")

    def ci_check(self, ws, stream=None):
        _check(_lib.ci_check(self._h, _ptr(ws), ws.numel(), _stream(stream)), "ci_check")


def ci_decode(h, h_parity, drop, ws, stream=None):
    B, k, d = h.shape
    _check(_lib.ci_decode(k, B, d, _ptr(h), _ptr(h_parity), _ptr(drop), _ptr(ws), ws.numel(),
                          _stream(stream)), "ci_decode")


def ci_decode_general(coef, h, h_parity, avail, ws, stream=None):
    r, k = coef.shape
    B, d = h.shape[0], h.shape[2]
    _check(_lib.ci_decode_general(k, r, B, d, _ptr(coef), _ptr(h), _ptr(h_parity), _ptr(avail), _ptr(ws),
                                  ws.numel(), _stream(stream)), "ci_decode_general")


def ci_online_update(k, est, state, task, value, ws, stream=None):
    """est [B][k][d] fp32, state [B] int64 (uint64 bits), task [B] int32, value [B][d] fp32."""
    B, d = est.shape[0], est.shape[2]
    _check(_lib.ci_online_update(k, B, d, _ptr(est), _ptr(state), _ptr(task), _ptr(value), _ptr(ws),
                                 ws.numel(), _stream(stream)), "ci_online_update")


def ci_make_drops(k, B, seed, drop, stream=None):
    _check(_lib.ci_make_drops(k, B, seed, _ptr(drop), _stream(stream)), "ci_make_drops")


def ci_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * CI_COMM_ID_BYTES)()
    _check(_lib.ci_comm_unique_id(buf), "ci_comm_unique_id")
    return bytes(buf)


class Comm:
    """Owns a ci_comm_t (include/codedinv.h "Communicator"): collective create / destroy."""

    def __init__(self, uid: bytes, nranks, rank, layout, max_B, d, device=0):
        assert len(uid) == CI_COMM_ID_BYTES
        self.nranks, self.rank, self.layout = nranks, rank, layout
        h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * CI_COMM_ID_BYTES).from_buffer_copy(uid)
        _check(_lib.ci_comm_create(buf, nranks, rank, layout, max_B, d, device, ctypes.byref(h)), "ci_comm_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ci_comm_destroy(self._h)
            self._h = None

    __del__ = close


def ci_last_error() -> str:
    return _lib.ci_last_error().decode()


# ---- instrumentation entry points (include/codedinv_testing.h)
def ci_test_prof_enable(enable=True):
    _check(_lib.ci_test_prof_enable(1 if enable else 0), "ci_test_prof_enable")


def ci_test_prof_read():
    """-> (ms[4], launches[4], flops[4]) per stage index since the last read."""
    ms = (ctypes.c_double * 4)()
    ln = (ctypes.c_int64 * 4)()
    fl = (ctypes.c_double * 4)()
    _check(_lib.ci_test_prof_read(ms, ln, fl), "ci_test_prof_read")
    return list(ms), list(ln), list(fl)


def ci_test_launch_count(reset=False):
    return int(_lib.ci_test_launch_count(1 if reset else 0))


def ci_test_rendezvous(uid: bytes, nranks, rank, payload: bytes):
    """-> list of every rank's payload (host-only shared-memory rendezvous of ci_comm_create)."""
    out = (ctypes.c_uint8 * (64 * nranks))()
    buf = (ctypes.c_uint8 * CI_COMM_ID_BYTES).from_buffer_copy(uid)
    pay = (ctypes.c_uint8 * max(len(payload), 1)).from_buffer_copy(payload or b"\0")
    _check(_lib.ci_test_rendezvous(buf, nranks, rank, pay, len(payload), out), "ci_test_rendezvous")
    raw = bytes(out)
    return [raw[64 * q:64 * q + len(payload)] for q in range(nranks)]


def ci_test_mean(h, m, stream=None):
    B, k, d = h.shape
    _check(_lib.ci_test_mean(k, B, d, _ptr(h), _ptr(m), _stream(stream)), "ci_test_mean")


PLAN_FIELDS = ["Wp", "G", "Cp", "Mp", "MC", "nch", "Nc2", "T", "I", "Rtot", "k1", "k2", "nslot",
               "slot_bytes", "smem", "blk_bytes", "nhd", "sstate", "est", "tmem_cols", "hst", "hc", "static",
               "ts", "nopad"]


def ci_test_plan(H, W, c, m, pm):
    """pm: 0 bf16, 1 f16x2, 2 f16x3 (CI_PREC_FP32)."""
    out = (ctypes.c_int64 * len(PLAN_FIELDS))()
    _check(_lib.ci_test_plan(H, W, c, m, int(pm), out), "ci_test_plan")
    return dict(zip(PLAN_FIELDS, list(out)))
