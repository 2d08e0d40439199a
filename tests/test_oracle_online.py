"""Pins of the online decoder oracle (oracle/online.py): SPEC.md:210-215
worked examples and exhaustive order enumeration against the batch decode."""
import itertools

import numpy as np
import pytest

import oracle
from oracle import online


def test_k2_trace_and_mains_only():
    rng = np.random.default_rng(0)
    v1, v2 = rng.standard_normal(6), rng.standard_normal(6)
    v3 = (v1 + v2) / 2
    st = online.run_events(2, [(2, v3), (0, v1)], 6)              # tasks 3 then 1 (1-based)
    assert st.finalized.all() and np.array_equal(st.est[1], 2 * v3 - v1)
    assert np.array_equal(st.est[0], v1)
    st = online.run_events(2, [(0, v1), (1, v2)], 6)              # parity never needed
    assert np.array_equal(st.est, [v1, v2])
    with pytest.raises(online.DuplicateTask):
        online.run_events(2, [(0, v1), (0, v1)], 6)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_every_order_of_every_k_subset_equals_batch_decode(k):
    """any permutation of any k of the k+1 events gives the batch-decode estimates;
    a late (k+1)-th event changes nothing."""
    rng = np.random.default_rng(k)
    d = 5
    H = rng.standard_normal((k, d))
    P = H.mean(0) + 1e-3 * rng.standard_normal(d)     # any parity value: the algebra is exact
    vals = [H[i] for i in range(k)] + [P]
    for S in itertools.combinations(range(k + 1), k):
        missing = [j for j in range(k) if j not in S]
        drop = np.array([missing[0] if missing else -1], np.int32)
        ref = oracle.decode(H[None], P[None], drop)[0]
        for order in itertools.permutations(S):
            st = online.run_events(k, [(j, vals[j]) for j in order], d)
            assert st.finalized.all()
            assert np.max(np.abs(st.est - ref)) < 1e-12
            late = [j for j in range(k + 1) if j not in S][0]
            before = st.est.copy()
            st.update(late, vals[late])
            assert np.array_equal(st.est, before)
