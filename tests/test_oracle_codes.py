"""Pins of the general (n, k) code oracle (oracle/codes.py).

Values are the paper's (Eq. 3, 567-590 multiple failures) or SPEC.md's worked
examples, closed-form 2x2 inverses, brute force over all k-subsets,
and the exact-recovery property of ideal encoding through an exactly invertible f."""
import itertools

import numpy as np
import pytest

import fixtures as fx
import oracle
from oracle import codes


def test_generator_examples():
    assert np.array_equal(codes.build_generator(3, 2, "uniform"), [[1, 0], [0, 1], [0.5, 0.5]])
    assert np.array_equal(codes.build_generator(2, 1, "uniform"), [[1], [1]])
    G = codes.build_generator(4, 2, "paper42")
    assert np.array_equal(G[2:], [[1 / 2, 1 / 2], [1 / 3, 2 / 3]])
    with pytest.raises(ValueError):
        codes.build_generator(5, 2, "uniform")
    with pytest.raises(ValueError):
        codes.build_generator(2, 3, "uniform")


def test_any_k_rows_checks():
    G = codes.build_generator(3, 2, "uniform")
    dets = [np.linalg.det(G[list(S)]) for S in itertools.combinations(range(3), 2)]
    assert np.allclose(dets, [1, 0.5, -0.5], atol=1e-15)
    assert codes.verify_any_k_rows(G)["ok"]
    bad = np.array([[1.0, 0], [0, 1], [0, 1]])
    rep = codes.verify_any_k_rows(bad)
    assert not rep["ok"] and rep["worst_subset"] == [1, 2]
    assert codes.verify_any_k_rows(codes.build_generator(5, 3, "gaussian", seed=7))["ok"]
    V = codes.build_generator(6, 4, "vandermonde")                      # all 15 subsets
    assert np.allclose(V[4:].sum(1), 1.0)
    n_ok = sum(abs(np.linalg.det(V[list(S)])) > 1e-12 for S in itertools.combinations(range(6), 4))
    assert n_ok == 15 and codes.verify_any_k_rows(V)["ok"]
    for n, k in ((4, 2), (6, 4), (7, 3)):
        assert codes.verify_any_k_rows(codes.build_generator(n, k, "vandermonde"))["ok"]


def test_subset_inverse_examples():
    U = codes.build_generator(3, 2, "uniform")
    assert np.allclose(codes.subset_inverse(U, [0, 2]), [[1, 0], [-1, 2]], atol=1e-15)   # Fig. 1
    assert np.array_equal(codes.subset_inverse(U, [0, 1]), np.eye(2))
    P = codes.build_generator(4, 2, "paper42")
    assert np.allclose(codes.subset_inverse(P, [2, 3]), [[4, -3], [-2, 3]], atol=1e-14)
    with pytest.raises(np.linalg.LinAlgError):
        codes.subset_inverse(np.array([[1.0, 0], [0, 1], [0, 1]]), [1, 2])


def test_decode_examples_and_uniform_special_case():
    rng = np.random.default_rng(0)
    v1, v2 = rng.standard_normal(5), rng.standard_normal(5)
    U = codes.build_generator(3, 2, "uniform")
    res = np.stack([v1, np.full(5, np.nan), (v1 + v2) / 2])[None]        # task 2 lost
    R = codes.decode(U, res, np.array([0b101]))
    assert np.allclose(R[0, 1], 2 * res[0, 2] - res[0, 0], atol=1e-15) and np.array_equal(R[0, 0], v1)
    full = np.stack([v1, v2, (v1 + v2) / 2])[None]
    assert np.allclose(codes.decode(U, full, np.array([0b111]))[0], [v1, v2], atol=0)
    # n = k + 1 uniform decode == the hot-path decode k P - sum_{i != j} H_i
    B, k, d = 6, 10, 33
    H = rng.standard_normal((B, k, d))
    Pp = H.mean(1)
    drop = rng.integers(0, k, B).astype(np.int32)
    G = codes.build_generator(k + 1, k, "uniform")
    res = np.concatenate([H, Pp[:, None]], 1)
    avail = np.array([((1 << (k + 1)) - 1) & ~(1 << int(j)) for j in drop])
    a = codes.decode(G, res, avail)
    b = oracle.decode(H, Pp, drop)
    assert np.max(np.abs(a - b)) < 1e-12
    # both data tasks lost, (4,2): recovered from the two parity rows alone
    P = codes.build_generator(4, 2, "paper42")
    res = np.stack([v1, v2, (v1 + v2) / 2, (v1 + 2 * v2) / 3])[None]
    assert np.allclose(codes.decode(P, res, np.array([0b1100]))[0], [v1, v2], atol=1e-14)


@pytest.mark.parametrize("n,k,scheme,arch", [(4, 2, "paper42", "T"), (6, 4, "vandermonde", "T"),
                                             (5, 3, "gaussian", "T"), (4, 2, "paper42", "TR")])
def test_ideal_encode_exact_recovery_every_subset(n, k, scheme, arch):
    """Ideal encoding makes f(x_{k+i}) = sum_j c_ij f(x_j), so decoding from ANY
    k tasks returns f(x_1..k) up to the inverse's rounding (coupling: exact inverse; residual:
    converged fixed point)."""
    arch = fx.ARCHS[arch]
    params = fx.make_weights(arch, 3)
    G = codes.build_generator(n, k, scheme, seed=1)
    subsets = list(itertools.combinations(range(n), k))
    B = len(subsets)
    x = fx.make_inputs(arch, B, k, 5)
    avail = np.array([sum(1 << i for i in S) for S in subsets])
    out = codes.serve_general(arch, params, x, G, avail)
    P_from_comb = out["P"] - out["comb"]                  # h(h^-1(comb)) - comb
    assert np.max(np.abs(P_from_comb)) < 1e-9 * max(1.0, np.max(np.abs(out["comb"])))
    err = np.max(np.abs(out["R"] - out["H"])) / np.max(np.abs(out["H"]))
    assert err < 1e-8, err
    # labels of decoded estimates equal the labels of the true features
    lg, lb = oracle.classify(arch, params, 0, out["H"].reshape(B * k, -1))
    assert np.array_equal(out["labels"][0].reshape(-1), lb)
