"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no convolution, coupling,
encode, decode or classifier).  It only defines

  * the architecture descriptors (workload definitions),
  * a counter-based splitmix64 generator,
  * the canonical flat parameter layout both sides parse independently,
  * seeded inputs x ~ U[0,1) and per-group drop indices.

Both the oracle (oracle/) and the CUDA path (paper_2106_06445_b200/) receive
the arrays produced here; neither imports the other.

Input recipe:
  - images x[B, k, C, H, W] fp32, i.i.d. U[0,1) (PAPER.md:393-426 use MNIST /
    CIFAR-10 images; values in [0,1) as ToTensor produces);
  - weights per SURVEY §8a "Weight init" with gain gamma = 0.1;
  - drop index per group j_b = (uint32)(splitmix64_at(seed, b) >> 32) % k:
    one uniformly random main worker lost per group ("one of the
    k workers", "randomly select an input x_a").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03


# --------------------------------------------------------------------------
# splitmix64 (counter based: the i-th output needs no previous state)
# --------------------------------------------------------------------------
def splitmix64_at(seed: int, idx):
    """(idx+1)-th output of splitmix64 seeded with `seed` (vectorised over idx).

    z_i = seed + (i+1)*GOLDEN;  z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
    z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + (idx + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def stream_seed(seed: int, tensor_id: int) -> int:
    return (seed ^ ((tensor_id * STREAM_MUL) & MASK64)) & MASK64


def uniform01(seed: int, tensor_id: int, n: int) -> np.ndarray:
    """n draws u = (z >> 11) * 2^-53 in [0,1), float64."""
    z = splitmix64_at(stream_seed(seed, tensor_id), np.arange(n, dtype=np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_f32(seed: int, tensor_id: int, n: int, lo: float, hi: float) -> np.ndarray:
    u = uniform01(seed, tensor_id, n)
    return (lo + (hi - lo) * u).astype(np.float32)


# --------------------------------------------------------------------------
# Architecture descriptors (readings Q1-Q6 in DESIGN.md)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Stage:
    squeeze_before: int  # 1: apply psi (space-to-depth r=2) before the blocks
    n_blocks: int
    mid: int             # hidden width m of F = conv3x3(c->m) -> act -> conv3x3(m->c)


@dataclass(frozen=True)
class Arch:
    name: str
    in_c: int
    in_h: int
    in_w: int
    stages: tuple
    act: str = "relu"            # "relu" | "elu" | "identity"
    first_orient: int = 0        # 0: block 0 does s_B += F(s_A); 1: s_A += F(s_B)
    heads: tuple = (10,)         # classes per linear head g_t
    gamma: float = 0.1           # gain on W2
    encoder: tuple = ()          # learned encoder (Arch E): (c1, mid); () = none
    # i-ResNet variant: "residual" blocks y = x + G(x) on the whole state,
    # each conv of G spectrally normalised to sqrt(lip) so Lip(G) <= lip < 1;
    # h^-1 runs fp_iters fixed-point updates per block (the stated N)
    block: str = "coupling"      # "coupling" | "residual"
    lip: float = 0.9
    fp_iters: int = 10

    def stage_shapes(self):
        """[(C, H, W, c, m, n_blocks)] of each stage after its squeeze; c = channels F acts on
        (C/2 for coupling, C for residual)."""
        C, H, W = self.in_c, self.in_h, self.in_w
        out = []
        for st in self.stages:
            if st.squeeze_before:
                C, H, W = C * 4, H // 2, W // 2
            out.append((C, H, W, C if self.block == "residual" else C // 2, st.mid, st.n_blocks))
        return out

    @property
    def d(self) -> int:
        C, H, W, *_ = self.stage_shapes()[-1]
        return C * H * W

    @property
    def act_id(self) -> int:
        return {"relu": 0, "elu": 1, "identity": 2}[self.act]

    @property
    def block_id(self) -> int:
        return {"coupling": 0, "residual": 1}[self.block]


ARCH_T = Arch("T", 3, 8, 8, (Stage(1, 2, 16),))
ARCH_M = Arch("M", 1, 28, 28, (Stage(1, 2, 32), Stage(1, 2, 64)))
ARCH_C = Arch("C", 3, 32, 32, (Stage(1, 9, 64), Stage(1, 9, 128), Stage(1, 9, 256)))
# Rotation pin (App. A.1) as three additive-coupling shears.
ARCH_R = Arch("R", 2, 1, 1, (Stage(0, 3, 1),), act="identity", first_orient=1, heads=())
# Arch C + light learned encoder (Arch E) + multitask heads fine 10 / coarse 2
# (PAPER.md:697-698): config C4.
ARCH_CE = Arch("CE", 3, 32, 32, ARCH_C.stages, heads=(10, 2), encoder=(16, 64))
# small encoder arch for fast oracle pins / GPU parity
ARCH_TE = Arch("TE", 3, 8, 8, ARCH_T.stages, heads=(10, 2), encoder=(4, 8))
# i-ResNet variant of Arch C (f1): channel plan 12/48/192, m = 64/128/256, ELU, L = 0.9,
# N = 10 fixed-point updates per block on the GPU (fp32-sufficient at L <= 0.9)
ARCH_CR = Arch("CR", 3, 32, 32, ARCH_C.stages, act="elu", block="residual")
ARCH_TR = Arch("TR", 3, 8, 8, (Stage(1, 2, 16),), act="elu", block="residual")
ARCHS = {a.name: a for a in (ARCH_T, ARCH_M, ARCH_C, ARCH_R, ARCH_CE, ARCH_TE, ARCH_CR, ARCH_TR)}


def linear_variant(arch: Arch) -> Arch:
    """Same shapes, identity activation (P1: h is linear when biases are 0)."""
    return Arch(arch.name + "lin", arch.in_c, arch.in_h, arch.in_w, arch.stages,
                act="identity", first_orient=arch.first_orient, heads=arch.heads,
                gamma=arch.gamma, encoder=arch.encoder, block=arch.block, lip=arch.lip,
                fp_iters=arch.fp_iters)


# --------------------------------------------------------------------------
# Canonical flat parameter layout
#   for stage s, block t:  W1[m][c][3][3], b1[m], W2[c][m][3][3], b2[c]
#   then per head:         Wg[classes][d], bg[classes]
#   then (learned encoder, Arch E):  E1.W[c1][in_c][3][3], E1.b[c1],
#        E2.W[mid][4c1][3][3], E2.b[mid], E3.W[4c1][mid][3][3], E3.b[4c1],
#        E4.W[in_c][c1][3][3], E4.b[in_c]
# --------------------------------------------------------------------------
def param_tensors(arch: Arch):
    """[(name, shape, lo, hi)] in canonical order."""
    out = []
    for s, (C, H, W, c, m, nb) in enumerate(arch.stage_shapes()):
        a1 = math.sqrt(6.0 / (9 * c))
        a2 = arch.gamma * math.sqrt(3.0 / (9 * m))
        for t in range(nb):
            out.append((f"s{s}b{t}.W1", (m, c, 3, 3), -a1, a1))
            out.append((f"s{s}b{t}.b1", (m,), -0.01, 0.01))
            out.append((f"s{s}b{t}.W2", (c, m, 3, 3), -a2, a2))
            out.append((f"s{s}b{t}.b2", (c,), -0.01, 0.01))
    d = arch.d
    ag = math.sqrt(3.0 / d)
    for i, ncls in enumerate(arch.heads):
        out.append((f"g{i}.W", (ncls, d), -ag, ag))
        out.append((f"g{i}.b", (ncls,), -0.01, 0.01))
    if arch.encoder:
        c1, mid = arch.encoder
        ci = arch.in_c
        for nm, co, cin, gain in (("E1", c1, ci, 6.0), ("E2", mid, 4 * c1, 6.0), ("E3", 4 * c1, mid, 6.0),
                                  ("E4", ci, c1, 3.0)):
            a = math.sqrt(gain / (9 * cin))
            out.append((f"{nm}.W", (co, cin, 3, 3), -a, a))
            out.append((f"{nm}.b", (co,), -0.01, 0.01))
    return out


def n_params(arch: Arch) -> int:
    return int(sum(np.prod(s) for _, s, _, _ in param_tensors(arch)))


def make_weights(arch: Arch, seed: int, zero_bias: bool = False) -> np.ndarray:
    """Flat fp32 parameter vector in canonical order (one splitmix64 stream per tensor).
    Residual archs: each block conv is then scaled to spectral norm sqrt(arch.lip)."""
    parts = []
    shapes = arch.stage_shapes()
    for tid, (name, shape, lo, hi) in enumerate(param_tensors(arch)):
        n = int(np.prod(shape))
        if zero_bias and (name.endswith(".b1") or name.endswith(".b2") or name.endswith(".b")):
            parts.append(np.zeros(n, np.float32))
            continue
        w = uniform_f32(seed, tid + 1, n, lo, hi)
        if arch.block == "residual" and name[0] == "s" and (name.endswith(".W1") or name.endswith(".W2")):
            _, H, W = shapes[int(name[1:name.index("b")])][:3]
            w4 = w.reshape(shape).astype(np.float64)
            sigma = conv_spectral_norm(w4, H, W, seed=seed * 1000003 + tid)
            w = (w4 * (math.sqrt(arch.lip) / sigma)).astype(np.float32).reshape(-1)
        parts.append(w)
    return np.concatenate(parts) if parts else np.zeros(0, np.float32)


# --------------------------------------------------------------------------
# Spectral normalisation (weight preparation of the i-ResNet variant, "bound
# each layer's Lipschitz constant by normalizing the weight matrix by its spectral norm";
# power iteration on conv / conv-transpose, 60 iterations).  This only
# shapes the frozen random weights both sides receive; it is not on the hot path.
# --------------------------------------------------------------------------
def _conv_nobias(x, w):
    """3x3 cross-correlation, zero padding 1: x [ci][H][W], w [co][ci][3][3] -> [co][H][W]."""
    ci, H, W = x.shape
    xp = np.zeros((ci, H + 2, W + 2))
    xp[:, 1:-1, 1:-1] = x
    out = np.zeros((w.shape[0], H, W))
    for u in range(3):
        for v in range(3):
            out += np.tensordot(w[:, :, u, v], xp[:, u:u + H, v:v + W], axes=1)
    return out


def _conv_adjoint(y, w):
    """Adjoint of _conv_nobias: y [co][H][W] -> [ci][H][W] (flipped, channel-swapped kernel)."""
    return _conv_nobias(y, np.ascontiguousarray(w.transpose(1, 0, 2, 3)[:, :, ::-1, ::-1]))


def conv_spectral_norm(w, H, W, iters=60, seed=0):
    """Largest singular value of the zero-padded 3x3 conv operator on an H x W grid."""
    v = uniform_f32(seed, 0, w.shape[1] * H * W, -1.0, 1.0).astype(np.float64).reshape(w.shape[1], H, W)
    v /= np.linalg.norm(v)
    sigma = 0.0
    for _ in range(iters):
        u = _conv_nobias(v, w)
        sigma = np.linalg.norm(u)
        u /= sigma
        v = _conv_adjoint(u, w)
        v /= np.linalg.norm(v)
    return float(np.linalg.norm(_conv_nobias(v, w)))


def split_params(arch: Arch, flat: np.ndarray) -> dict:
    """Views into the flat vector by canonical name (layout bookkeeping only)."""
    out, off = {}, 0
    for name, shape, _, _ in param_tensors(arch):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    assert off == flat.size
    return out


def rotation_params(theta: float, seed: int = 7) -> np.ndarray:
    """ARCH_R parameters realising R(theta) as shears A,B,A.

    Centre taps carry the shear; the 8 off-centre taps are random and must be
    ignored by zero padding of the 1x1 image.
    """
    flat = make_weights(ARCH_R, seed)
    p = split_params(ARCH_R, flat)
    shear = [-math.tan(theta / 2), math.sin(theta), -math.tan(theta / 2)]
    for t in range(3):
        p[f"s0b{t}.W1"][0, 0, 1, 1] = 1.0
        p[f"s0b{t}.b1"][:] = 0.0
        p[f"s0b{t}.W2"][0, 0, 1, 1] = shear[t]
        p[f"s0b{t}.b2"][:] = 0.0
    return flat


# --------------------------------------------------------------------------
# Inputs and drops
# --------------------------------------------------------------------------
def make_inputs(arch: Arch, B: int, k: int, seed: int) -> np.ndarray:
    n = B * k * arch.in_c * arch.in_h * arch.in_w
    return uniform_f32(seed, 0, n, 0.0, 1.0).reshape(B, k, arch.in_c, arch.in_h, arch.in_w)


def make_inputs_slice(arch: Arch, b0: int, b1: int, k: int, seed: int) -> np.ndarray:
    """Groups [b0, b1) of make_inputs(arch, B, k, seed) for any B >= b1, generated directly
    (counter-based stream: element e of the global tensor is splitmix64_at(stream, e))."""
    per = k * arch.in_c * arch.in_h * arch.in_w
    idx = np.arange(b0 * per, b1 * per, dtype=np.uint64)
    z = splitmix64_at(stream_seed(seed, 0), idx)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return u.astype(np.float32).reshape(b1 - b0, k, arch.in_c, arch.in_h, arch.in_w)


def make_drops_slice(b0: int, b1: int, k: int, seed: int) -> np.ndarray:
    z = splitmix64_at(seed & MASK64, np.arange(b0, b1, dtype=np.uint64))
    return ((z >> np.uint64(32)) % np.uint64(k)).astype(np.int32)


def shard(rank: int, world: int, groups_per_rank: int):
    """Group-sharded data parallelism: rank r serves global groups [r*B, (r+1)*B)."""
    assert 0 <= rank < world
    return rank * groups_per_rank, (rank + 1) * groups_per_rank


def make_drops(B: int, k: int, seed: int) -> np.ndarray:
    """j_b = (uint32)(splitmix64_at(seed, b) >> 32) % k, int32[B]."""
    z = splitmix64_at(seed & MASK64, np.arange(B, dtype=np.uint64))
    return ((z >> np.uint64(32)) % np.uint64(k)).astype(np.int32)


def group_of(q, k: int):
    """Query q -> (group b, slot i) = (q div k, q mod k)."""
    q = np.asarray(q, dtype=np.int64)
    return q // k, q % k


# --------------------------------------------------------------------------
# Named workloads = BASELINE.json configs
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    arch: Arch
    k: int
    B: int
    seed_w: int
    seed_x: int
    seed_drop: int
    note: str = ""


CONFIGS = {
    "C1": Config("C1", ARCH_T, 2, 4, 11, 1, 101, "k=2 tiny 2-block net on 3x8x8, 4 groups"),
    "C2": Config("C2", ARCH_M, 4, 256, 12, 2, 102, "k=4 MNIST-shaped 1x28x28, 256 groups"),
    "C3": Config("C3", ARCH_C, 10, 1024, 13, 3, 103,
                 "k=10 CIFAR-shaped 3x32x32 full-depth h, exact h^-1 parity encode, 1024 groups"),
    "C4": Config("C4", ARCH_CE, 10, 1024, 14, 4, 104,
                 "k=10 CIFAR-shaped, light learned encoder replaces h^-1, multitask heads 10 + 2"),
    "C5": Config("C5", ARCH_CE, 7, 1024, 15, 5, 105,
                 "k=7 main + 1 parity worker, one per GPU (8 GPUs), exact or learned encode, "
                 "decode as a masked reduction over workers"),
    # not a BASELINE config: the i-ResNet variant at C3's shape
    "C3R": Config("C3R", ARCH_CR, 10, 1024, 16, 6, 106,
                  "f1: C3 with i-ResNet residual blocks (12/48/192 channels, ELU, Lip 0.9); "
                  "exact encode h^-1 by 10 fixed-point updates per block"),
}


def arch_summary(arch: Arch) -> str:
    """One-line description of an arch for bench JSON lines."""
    kind = "i-ResNet residual" if arch.block == "residual" else "additive-coupling"
    sh = arch.stage_shapes()
    s = (f"{arch.name}: {len(sh)} stages x {'/'.join(str(x[5]) for x in sh)} {kind} blocks "
         f"(c={'/'.join(str(x[3]) for x in sh)}, m={'/'.join(str(x[4]) for x in sh)}, {arch.act})")
    if arch.block == "residual":
        s += f", h^-1 = {arch.fp_iters} fixed-point updates/block"
    if arch.encoder:
        s += f", learned encoder {arch.encoder}"
    return s
