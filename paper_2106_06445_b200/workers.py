"""Bootstrap of the worker-partitioned coded serving (config C5) for torch.distributed jobs.

The paper's partition (Fig. 2, 665-668: one worker per instance): rank r < k is
main worker r (slot r of every group), rank k is the parity worker and hosts the encoder
(PAPER.md:284-289, 667).  The exchange steps (X2 mean for the exact encode, X4 decode) run
inside libcodedinv as fused kernels over peer memory (include/codedinv.h "Communicator");
this module only broadcasts the communicator id and shapes the per-rank buffers -- argument
marshalling, no arithmetic.
"""
from __future__ import annotations

from paper_2106_06445_b200 import codedinv as ci


def make_comm(dist, layout, max_B, d, device=0):
    """Collective: rank 0 draws the id, torch.distributed broadcasts it, every rank maps the
    others' windows (ci_comm_create)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    box = [ci.ci_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return ci.Comm(box[0], world, rank, layout, max_B, d, device)


class WorkerBuffers:
    """Device outputs of one rank of a CI_SHARD_WORKERS serve (shapes of ci_serve_group)."""

    def __init__(self, model, k, B, device):
        import torch
        a = model.arch
        self.B, self.Bp = B, (B + k) // (k + 1)
        self.h = torch.empty(B, model.d, device=device)
        self.dec = torch.empty(self.Bp, model.d, device=device)
        self.xp = torch.empty(B, a.in_c, a.in_h, a.in_w, device=device)
        rows = B + self.Bp
        self.logits = torch.empty(max(rows * sum(a.heads), 1), device=device)
        self.labels = torch.empty(max(rows * len(a.heads), 1), dtype=torch.int32, device=device)
        self.ws = model.workspace(k, B)

    def head(self, t, heads):
        """(own-slot logits [B][C], decoded-partition logits [Bp][C], labels alike) of head t."""
        rows = self.B + self.Bp
        lo = rows * sum(heads[:t])
        lg = self.logits[lo:lo + rows * heads[t]].view(rows, heads[t])
        lb = self.labels[t * rows:(t + 1) * rows]
        return lg[:self.B], lg[self.B:], lb[:self.B], lb[self.B:]


def serve_worker(model, comm, x, drop, bufs, learned=False, stream=None):
    """One collective serve call: x = this rank's slot [B, C, H, W] (main ranks), the k slots
    [B, k, C, H, W] (parity rank, learned mode) or None (parity rank, exact mode)."""
    model.ci_serve_group(x, drop, bufs.h, bufs.dec, bufs.ws, x_parity=bufs.xp, logits=bufs.logits,
                         labels=bufs.labels, learned=learned, comm=comm, stream=stream)
