"""Worker-partitioned coded serving (config C5): the paper's partition, one worker per GPU.

PAPER.md:201-214 (Fig. 2): k main workers each compute f on one query of the group, n-k = 1
parity worker computes f on the encoded query; the front end decodes from any k results
(MPI workers on EC2).  Here: rank w < k is main worker w (slot w of every
group), rank k is the parity worker and hosts the encoder.

Exchange steps (torch.distributed; NCCL over NVLink on the GPUs):
  X2 (exact encode)  : reduce(sum) of (1/k) h_w onto the parity rank -> mean; then h^-1, h
  X3 (learned encode): the parity rank holds all k inputs of its groups (front-end delivery)
  X4 (decode)        : decode is linear, so it rides a reduction: every worker contributes
                       coef_w[b] * f_w[b] (coef -1 / 0 / +k, ci_worker_coef) and a
                       reduce-scatter over group partitions leaves rank p with the decoded
                       features of the lost slot for groups [p B/n, (p+1) B/n).
Drops are simulated by masking (coefficient 0): collectives need every rank, so this measures
throughput, not straggler latency.

The per-rank compute is injected (GpuCompute drives the C ABI; tests inject a CPU stand-in),
so the orchestration logic is exercised with gloo on CPU (tests/test_multiproc.py).
"""
from __future__ import annotations

COEF_DECODE, COEF_MEAN = 0, 1


class GpuCompute:
    """Per-rank compute through libcodedinv (device tensors, current torch stream)."""

    def __init__(self, model, k, B):
        import torch
        from paper_2106_06445_b200 import codedinv as ci
        self.ci, self.torch, self.model, self.k, self.B = ci, torch, model, k, B
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.ws = model.workspace(k, B)
        self.d = model.d
        a = model.arch
        self.img = (a.in_c, a.in_h, a.in_w)

    def empty(self, *shape):
        return self.torch.empty(*shape, device=self.dev)

    def zeros(self, *shape):
        return self.torch.zeros(*shape, device=self.dev)

    def forward_h(self, x):
        h = self.empty(x.shape[0], self.d)
        self.model.ci_forward_h(x, h, self.ws)
        return h

    def inverse_h(self, h):
        x = self.empty(h.shape[0], *self.img)
        self.model.ci_inverse_h(h, x, self.ws)
        return x

    def encode_learned(self, x_all):
        xp = self.empty(x_all.shape[0], *self.img)
        self.model.ci_encode(None, xp, self.ws, x=x_all, learned=True)
        return xp

    def coef(self, kind, worker, drop):
        c = self.empty(drop.shape[0])
        self.ci.ci_worker_coef(kind, self.k, drop.shape[0], worker, drop, c)
        return c

    def combine(self, f, coef):
        out = self.empty(*f.shape)
        self.ci.ci_combine(f, coef, out)
        return out

    def classify(self, head, z):
        C = self.model.arch.heads[head]
        logits = self.empty(z.shape[0], C)
        labels = self.torch.empty(z.shape[0], dtype=self.torch.int32, device=self.dev)
        self.model.ci_classify(head, z, logits, labels)
        return logits, labels


def _reduce_scatter(dist, out, inp, rank, world):
    """Sum over ranks, rank p keeps rows [p*len(out), (p+1)*len(out)).  NCCL: one
    reduce-scatter; backends without it (gloo, CPU tests): all-reduce and slice."""
    if dist.get_backend() == "nccl":
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM)
    else:
        full = inp.clone()
        dist.all_reduce(full, op=dist.ReduceOp.SUM)
        n = out.shape[0]
        out.copy_(full[rank * n:(rank + 1) * n])


def serve_workers(compute, dist, rank, world, k, drop, x_slot=None, x_all=None, learned=False):
    """One coded serving step on this rank.

    rank < k : main worker `rank`; x_slot [B, C, H, W] = slot `rank` of every group.
    rank == k: parity worker; x_all [B, k, C, H, W] (learned mode only).
    Returns {"f": this worker's features [B, d] (h(x_slot) or h(x_p)),
             "decoded": [B/world, d] decoded lost-slot features of this rank's group partition,
             "logits": [heads] of (own-slot logits [B, C_t]) (main ranks),
             "logits_decoded": [heads] of decoded-partition logits [B/world, C_t]}."""
    assert world == k + 1, "worker partition needs one rank per worker (n = k + 1)"
    B = drop.shape[0]
    assert B % world == 0, "groups must split evenly over the reduce-scatter partitions"
    parity = rank == k
    # (1) h on this worker's query
    f = None if parity else compute.forward_h(x_slot)
    # (2) encode
    if learned:
        xp = compute.encode_learned(x_all) if parity else None                       # X3
    else:
        contrib = compute.zeros(B, compute.d) if parity else compute.combine(f, compute.coef(COEF_MEAN, rank, drop))
        dist.reduce(contrib, dst=k, op=dist.ReduceOp.SUM)                              # X2
        xp = compute.inverse_h(contrib) if parity else None
    # (3) h on the parity query
    if parity:
        f = compute.forward_h(xp)
    # (4) decode: masked reduce-scatter of coef_w * f_w over group partitions           # X4
    contrib = compute.combine(f, compute.coef(COEF_DECODE, rank, drop))
    decoded = compute.empty(B // world, compute.d)
    _reduce_scatter(dist, decoded, contrib, rank, world)
    # (5) heads: own-slot features (main ranks) and the decoded partition (every rank)
    out = {"f": f, "decoded": decoded, "logits": [], "logits_decoded": []}
    for t in range(len(compute.model.arch.heads)):
        if not parity:
            out["logits"].append(compute.classify(t, f)[0])
        out["logits_decoded"].append(compute.classify(t, decoded)[0])
    return out
