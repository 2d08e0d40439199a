"""General (n, k) codes for Coded-InvNet -- f64 numpy oracle.

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py): imported by tests/ and bench.py's
cpu_baseline legs, never by the product package.

What is computed, with the passage each step follows:
  generator G (n x k) ...... systematic: first k rows = I_k, parity rows c_{i,j} (PAPER.md:
                             216-238, Eq. 3); schemes: Uniform n = k+1, c = 1/k;
                             PaperMulti42 rows [1/2, 1/2], [1/3, 2/3];
                             Vandermonde rows (a_i^0 .. a_i^{k-1}) / sum with nodes a_i = i + 2
                             (reading R-f3a); GaussianRandom i.i.d. N(0,1)
  decodability ............. any k rows full rank, checked on every k-subset
                             by the scaled determinant
  subset inverse ........... inv(G_S) (Eq. 2 "simply multiply the inverse")
  encode ................... x_{k+i} = h^-1(sum_j c_{i,j} h(x_j)), i = 1..n-k
  decode ................... S = the k smallest available task indices (reading R-f3b);
                             (f^(x_1) .. f^(x_k)) = inv(G_S) [f(x_s)]_{s in S}
"""
from __future__ import annotations

import itertools

import numpy as np

from . import classify, forward_h, inverse_h

SING_TOL = 1e-9


def build_generator(n: int, k: int, scheme: str = "uniform", seed: int = 0) -> np.ndarray:
    """G [n][k] f64."""
    if not 1 <= k <= n:
        raise ValueError("need 1 <= k <= n")
    G = np.zeros((n, k))
    G[:k] = np.eye(k)
    r = n - k
    if scheme == "uniform":
        if r != 1:
            raise ValueError("Uniform needs n = k + 1")
        G[k] = 1.0 / k
    elif scheme == "paper42":
        if (n, k) != (4, 2):
            raise ValueError("PaperMulti42 needs (n, k) = (4, 2)")
        G[2] = [1 / 2, 1 / 2]
        G[3] = [1 / 3, 2 / 3]
    elif scheme == "vandermonde":
        for i in range(r):
            row = (i + 2.0) ** np.arange(k)
            G[k + i] = row / row.sum()
    elif scheme == "gaussian":
        rng = np.random.default_rng(seed)
        for _ in range(100):
            G[k:] = rng.standard_normal((r, k))
            if verify_any_k_rows(G)["ok"]:
                break
        else:
            raise RuntimeError("ValidationFailed")
    else:
        raise ValueError(scheme)
    return G


def scaled_det(M: np.ndarray) -> float:
    """|det| after scaling every row to unit 2-norm."""
    norms = np.linalg.norm(M, axis=1)
    if np.any(norms == 0):
        return 0.0
    return abs(float(np.linalg.det(M / norms[:, None])))


def verify_any_k_rows(G: np.ndarray) -> dict:
    n, k = G.shape
    worst, margin = None, np.inf
    for S in itertools.combinations(range(n), k):
        d = scaled_det(G[list(S)])
        if d < margin:
            worst, margin = list(S), d
    return {"ok": margin > SING_TOL, "worst_subset": worst, "worst_margin": margin}


def subset_inverse(G: np.ndarray, subset) -> np.ndarray:
    M = G[list(subset)]
    if scaled_det(M) <= SING_TOL:
        raise np.linalg.LinAlgError("SingularSubset")
    return np.linalg.inv(M)


def decode_subset(avail: int, n: int, k: int):
    """k smallest available task indices (bit i of avail = task i arrived), or None."""
    S = [i for i in range(n) if (avail >> i) & 1][:k]
    return S if len(S) == k else None


def decode(G: np.ndarray, results: np.ndarray, avail) -> np.ndarray:
    """results [B][n][d] (unavailable rows ignored), avail [B] bitmasks -> [B][k][d]
    estimates of f(x_1..k)."""
    n, k = G.shape
    B = results.shape[0]
    out = np.empty((B, k, results.shape[2]))
    for b in range(B):
        S = decode_subset(int(avail[b]), n, k)
        if S is None:
            raise ValueError(f"group {b}: fewer than k results")
        out[b] = subset_inverse(G, S) @ results[b, S]
    return out


def encode(arch, params, H: np.ndarray, G: np.ndarray, nthreads=None, fp_iters=0):
    """H [B][k][d] -> (combinations [B][r][d], x_parity [B][r][C][H][W])."""
    n, k = G.shape
    B, d = H.shape[0], H.shape[2]
    comb = np.einsum("ij,bjd->bid", G[k:], H)
    xp = inverse_h(arch, params, comb.reshape(-1, d), nthreads, fp_iters=fp_iters)
    return comb, xp.reshape(B, n - k, arch.in_c, arch.in_h, arch.in_w)


def serve_general(arch, params, x, G, avail, nthreads=None, fp_iters=0):
    """Whole coded path for an (n, k) code: h on the k main queries, n-k parity queries
    encoded and run through h, decode from the k smallest available tasks, heads on the
    decoded estimates.  x [B][k][C][H][W]."""
    n, k = G.shape
    B = x.shape[0]
    d = arch.d
    Hm = forward_h(arch, params, x.reshape(B * k, *x.shape[2:]), nthreads).reshape(B, k, d)
    comb, xp = encode(arch, params, Hm, G, nthreads, fp_iters)
    P = forward_h(arch, params, xp.reshape(B * (n - k), *xp.shape[2:]), nthreads).reshape(B, n - k, d)
    R = decode(G, np.concatenate([Hm, P], 1), avail)
    out = dict(H=Hm, comb=comb, xp=xp, P=P, R=R, logits=[], labels=[])
    for t in range(len(arch.heads)):
        lg, lb = classify(arch, params, t, R.reshape(B * k, d))
        out["logits"].append(lg.reshape(B, k, -1))
        out["labels"].append(lb.reshape(B, k))
    return out
