import sys, numpy as np, torch
sys.path.insert(0, '.')
import fixtures as fx, oracle
from paper_2106_06445_b200 import codedinv as ci
arch = fx.ARCH_TE; k = 3; Q = 6
params = fx.make_weights(arch, 14)
x = fx.make_inputs(arch, Q, k, 8)
strag = np.array([0, 1, 2, -1, 0, 1], np.int32)
m = ci.Model(arch, params, "fp32")
ref = oracle.serve_group(arch, params, x, strag, learned=True)
for delay in (0, 30_000_000):
  for inflight in (1, 4):
    feats = torch.empty(Q, k, arch.d, device="cuda")
    logits = torch.empty(Q * k * 12, device="cuda"); labels = torch.empty(Q * k * 2, dtype=torch.int32, device="cuda")
    rec = torch.zeros(Q, 4, dtype=torch.int64, device="cuda")
    ws = m.workspace_first_k(k, inflight)
    m.ci_serve_first_k(torch.from_numpy(x).cuda(), strag, delay, feats, logits, labels, rec, ws, max_inflight=inflight)
    torch.cuda.synchronize()
    F = feats.cpu().numpy(); r = rec.cpu().numpy()
    print("delay", delay, "inflight", inflight)
    for q in range(Q):
        errs = [float(np.max(np.abs(F[q, i] - ref["R"][q, i])) / np.max(np.abs(ref["R"][q, i]))) for i in range(k)]
        errH = [float(np.max(np.abs(F[q, i] - ref["H"][q, i])) / np.max(np.abs(ref["H"][q, i]))) for i in range(k)]
        print(q, strag[q], "lat ms %.3f" % (r[q, 0] / 1e6), "mask", bin(r[q, 3] & 0xffffffff), "deg", r[q, 3] >> 32,
              "errR", ["%.1e" % e for e in errs], "errH", ["%.1e" % e for e in errH])
# the parity result itself: single-GPU learned serve
xt = torch.from_numpy(x).cuda(); dt = torch.from_numpy(np.maximum(strag, -1)).cuda()
h = torch.empty(Q, k, arch.d, device="cuda"); p = torch.empty(Q, arch.d, device="cuda")
ws = m.workspace(k, Q)
m.ci_serve_group(xt, dt, h, p, ws, learned=True)
torch.cuda.synchronize()
print("single-GPU P err", float(np.max(np.abs(p.cpu().numpy() - ref["P"]))))
import os
print("CUDA_DEVICE_MAX_CONNECTIONS", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"))
Q = 40
x = fx.make_inputs(arch, Q, k, 9)
strag = np.random.default_rng(1).integers(0, k, Q).astype(np.int32)
for inflight in (4, 8, 16):
    feats = torch.empty(Q, k, arch.d, device="cuda")
    logits = torch.empty(Q * k * 12, device="cuda"); labels = torch.empty(Q * k * 2, dtype=torch.int32, device="cuda")
    rec = torch.zeros(Q, 4, dtype=torch.int64, device="cuda")
    ws = m.workspace_first_k(k, inflight)
    m.ci_serve_first_k(torch.from_numpy(x).cuda(), strag, 30_000_000, feats, logits, labels, rec, ws, max_inflight=inflight)
    torch.cuda.synchronize()
    r = rec.cpu().numpy()
    print("inflight", inflight, "lat ms p50 %.3f max %.3f" % (np.median(r[:, 0]) / 1e6, r[:, 0].max() / 1e6), "degraded", (r[:, 3] >> 32).mean())
