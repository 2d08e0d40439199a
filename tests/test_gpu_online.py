"""GPU online decoding (ci_online_update; App. C) against the
oracle decoder state machine (oracle/online.py) and the batch decode."""
import itertools

import numpy as np
import pytest

import oracle
from oracle import online

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_06445_b200 import codedinv
    return codedinv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_waves(ci, k, orders, vals, d):
    """orders[b] = sequence of tasks for group b; vals [B][k+1][d]."""
    B = len(orders)
    est = torch.zeros(B, k, d, device="cuda")
    state = torch.zeros(B, dtype=torch.int64, device="cuda")
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    nw = max(len(o) for o in orders)
    for w in range(nw):
        task = np.array([o[w] if w < len(o) else -1 for o in orders], np.int32)
        value = np.stack([vals[b, t] if t >= 0 else np.zeros(d, np.float32) for b, t in enumerate(task)])
        ci.ci_online_update(k, est, state, dev(task), dev(value.astype(np.float32)), ws)
    torch.cuda.synchronize()
    return est.cpu().numpy(), state.cpu().numpy(), ws


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("d", [8, 6])      # float4 and scalar paths
def test_online_every_order_bit_exact(ci, k, d):
    """Integer-valued results: every order of every event sequence (k of k+1 tasks, plus the
    late one) is bit-exact with the oracle state machine."""
    rng = np.random.default_rng(k * 10 + d)
    orders = []
    for S in itertools.combinations(range(k + 1), k):
        late = [j for j in range(k + 1) if j not in S]
        for perm in itertools.permutations(S):
            orders.append(list(perm) + late)
    B = len(orders)
    vals = rng.integers(-512, 512, size=(B, k + 1, d)).astype(np.float32)
    est, state, _ = run_waves(ci, k, orders, vals, d)
    for b, o in enumerate(orders):
        st = online.run_events(k, [(j, vals[b, j].astype(np.float64)) for j in o], d)
        assert np.array_equal(est[b].astype(np.float64), st.est), (b, o)
        R = int(state[b]) & 0xFFFFFFFF
        F = (int(state[b]) >> 32) & 0xFFFFFFFF
        assert R == (1 << (k + 1)) - 1 and F == (1 << k) - 1


def test_online_equals_batch_decode_c3_size(ci):
    """k = 10, d = 3072, 512 groups, random arrival order of all 11 tasks; after the k-th event
    the estimates equal the batch decode k P - sum (same fp32 values up to rounding order)."""
    k, B, d = 10, 512, 3072
    rng = np.random.default_rng(3)
    H = rng.standard_normal((B, k, d)).astype(np.float32)
    P = H.mean(1).astype(np.float32)
    vals = np.concatenate([H, P[:, None]], 1)
    orders = [list(rng.permutation(k + 1)) for _ in range(B)]
    first_k = [o[:k] for o in orders]
    est, state, _ = run_waves(ci, k, first_k, vals, d)
    drop = np.array([[j for j in range(k) if j not in o][0] if k in o else -1 for o in first_k], np.int32)
    ref = oracle.decode(H.astype(np.float64), P.astype(np.float64), drop)
    err = np.max(np.abs(est - ref)) / np.max(np.abs(ref))
    assert err < 1e-5, err
    # the late event changes nothing
    est2, _, _ = run_waves(ci, k, orders, vals, d)
    assert np.array_equal(est, est2)


def test_online_duplicate_task_flag(ci):
    k, d = 3, 8
    vals = np.ones((2, k + 1, d), np.float32)
    est, state, ws = run_waves(ci, k, [[0, 0], [1, 2]], vals, d)
    assert int(ws[:4].view(torch.int32).item()) == 1
    assert np.array_equal(est[0, 0], vals[0, 0])
