"""GPU tests of the first-k gated serving harness (App. C
PAPER.md:938-952): k main workers + the parity worker on their own
streams, one main worker per query delayed, online decoding on arrival.  Checked against the
f64 oracle: the k recovered features of every query (the straggler's slot decoded from the
parity when it is late) and the heads; first-k gating (coded latency never waits
for the straggler); the uncoded arm waits for it."""
import numpy as np
import pytest

import fixtures as fx
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-3


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


def run(ci, m, arch, x, strag, delay_ns, uncoded, inflight=8):
    Q, k = x.shape[:2]
    feats = torch.empty(Q, k, arch.d, device="cuda")
    logits = torch.empty(Q * k * sum(arch.heads), device="cuda")
    labels = torch.empty(Q * k * len(arch.heads), dtype=torch.int32, device="cuda")
    rec = torch.zeros(Q, 4, dtype=torch.int64, device="cuda")
    ws = m.workspace_first_k(k, inflight)
    m.ci_serve_first_k(torch.from_numpy(x).cuda(), strag, delay_ns, feats, logits, labels, rec, ws,
                       max_inflight=inflight, uncoded=uncoded)
    torch.cuda.synchronize()
    return feats.cpu().numpy(), logits.cpu().numpy(), labels.cpu().numpy(), rec.cpu().numpy()


@pytest.mark.parametrize("k,Q", [(3, 24), (10, 12)])
def test_first_k_coded_and_uncoded_vs_oracle(ci, k, Q):
    arch = fx.ARCH_TE if k == 3 else fx.ARCH_CE
    params = fx.make_weights(arch, 14)
    x = fx.make_inputs(arch, Q, k, 8)
    rng = np.random.default_rng(k)
    strag = rng.integers(0, k, Q).astype(np.int32)
    strag[::5] = -1                                  # some queries without a straggler
    delay = 30_000_000                               # 30 ms
    m = ci.Model(arch, params, "fp32")
    ref = oracle.serve_group(arch, params, x, strag, learned=True)   # drop = the straggler's slot
    for uncoded in (False, True):
        F, L, lab, rec = run(ci, m, arch, x, strag, delay, uncoded)
        lat, mask, degraded = rec[:, 0], rec[:, 3] & 0xFFFFFFFF, rec[:, 3] >> 32
        has = strag >= 0
        if uncoded:   # waits for every main worker: the straggler's true result
            assert relerr(F, ref["H"]) < TOL
            assert np.all(lat[has] >= delay) and np.all(degraded == 0)
            assert np.all(mask == (1 << k) - 1)
        else:         # first k: the parity replaces the straggler; never waits for it
            assert relerr(F, ref["R"]) < TOL
            assert np.all(lat < delay), lat.max()
            for q in np.nonzero(has)[0]:
                assert not (mask[q] >> strag[q]) & 1 and (mask[q] >> k) & 1 and degraded[q] == 1
            assert np.all([bin(int(v)).count("1") == k for v in mask])
        lo = 0
        for t, C in enumerate(arch.heads):
            lg = L[lo:lo + Q * k * C].reshape(Q, k, C)
            want = ref["logits_n" if uncoded else "logits"][t]
            assert relerr(lg, want) < TOL
            lb = lab[t * Q * k:(t + 1) * Q * k].reshape(Q, k)
            assert np.array_equal(lb, np.argmax(lg, -1))
            lo += Q * k * C
        print(f"[first-k k={k} {'uncoded' if uncoded else 'coded'}] latency p50 {np.median(lat) / 1e6:.3f} ms "
              f"max {lat.max() / 1e6:.3f} ms, update {np.median(rec[:, 1]) / 1e3:.1f} us, heads "
              f"{np.median(rec[:, 2]) / 1e3:.1f} us")


def test_first_k_needs_the_learned_encoder(ci):
    arch = fx.ARCH_T
    m = ci.Model(arch, fx.make_weights(arch, 11), "fp32")
    x = fx.make_inputs(arch, 2, 2, 1)
    with pytest.raises(ci.CiError) as e:   # no encoder: the parity worker cannot encode
        run(ci, m, arch, x, np.array([0, 1], np.int32), 1000, uncoded=False)
    assert e.value.status == ci.CI_ERR_UNSUPPORTED
