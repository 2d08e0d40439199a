"""GPU tests of the worker-partitioned serve (config C5 shape: one process per worker, k + 1
ranks) through the C ABI: ci_comm_create + ci_serve_group
with a CI_SHARD_WORKERS communicator.  All ranks run on the one GPU of the test box (the
peer-memory exchange works the same between processes of one GPU and across NVLink), two
serve calls per run (the second exercises the epoch protocol: publish after every peer is done
with the previous call).  Checked against
  * the f64 oracle (oracle.serve_group on all k slots): each main rank's h(x_r), the parity
    rank's x_p and h(x_p), the decoded lost-slot features of every rank's share of the groups,
    the heads on both, all within 1e-3 (fp32 precision);
  * the single-process ci_serve_group on the same inputs, bit for bit: the fused peer-memory
    mean / decode use the same fp32 summation order as k_mean / k_decode.
"""
import os
import socket

import numpy as np
import pytest

import fixtures as fx
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, arch_name, k, B, learned, seeds, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2106_06445_b200 import codedinv as ci
    from paper_2106_06445_b200.workers import WorkerBuffers, make_comm, serve_worker
    arch = fx.ARCHS[arch_name]
    model = ci.Model(arch, fx.make_weights(arch, 15), "fp32")
    comm = make_comm(dist, ci.CI_SHARD_WORKERS, B, model.d)
    bufs = WorkerBuffers(model, k, B, "cuda")
    for call, (sx, sd) in enumerate(seeds):
        x = fx.make_inputs(arch, B, k, sx)
        drop = fx.make_drops(B, k, sd)
        drop[1] = -1                                     # a group without a loss
        dt = torch.from_numpy(drop).cuda()
        if rank < k:
            xin = torch.from_numpy(np.ascontiguousarray(x[:, rank])).cuda()
        else:
            xin = torch.from_numpy(x).cuda() if learned else None
        serve_worker(model, comm, xin, dt, bufs, learned=learned)
        torch.cuda.synchronize()
        model.ci_check(bufs.ws)
        np.savez(os.path.join(out_dir, f"r{rank}_c{call}.npz"), h=bufs.h.cpu().numpy(), dec=bufs.dec.cpu().numpy(),
                 xp=bufs.xp.cpu().numpy(), logits=bufs.logits.cpu().numpy(), labels=bufs.labels.cpu().numpy())
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def relerr(a, ref):
    a = np.asarray(a, np.float64).reshape(-1, np.shape(ref)[-1])
    r = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


@pytest.mark.parametrize("arch_name,k,B,learned", [("T", 2, 7, False), ("TE", 3, 10, True), ("CE", 7, 20, False),
                                                   ("CE", 7, 20, True)])
def test_worker_partition_vs_oracle_and_single_gpu(tmp_path, arch_name, k, B, learned):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world = k + 1
    seeds = [(5, 105), (6, 106)]
    mp.spawn(_rank, args=(world, _free_port(), arch_name, k, B, learned, seeds, str(tmp_path)), nprocs=world,
             join=True)
    from paper_2106_06445_b200 import codedinv as ci
    arch = fx.ARCHS[arch_name]
    params = fx.make_weights(arch, 15)
    single = ci.Model(arch, params, "fp32")
    Bp = (B + k) // (k + 1)
    heads = arch.heads
    for call, (sx, sd) in enumerate(seeds):
        x = fx.make_inputs(arch, B, k, sx)
        drop = fx.make_drops(B, k, sd)
        drop[1] = -1
        ref = oracle.serve_group(arch, params, x, drop, learned=learned)
        # single-process path on the same inputs
        xt, dt = torch.from_numpy(x).cuda(), torch.from_numpy(drop).cuda()
        hs = torch.empty(B, k, arch.d, device="cuda")
        ps = torch.empty(B, arch.d, device="cuda")
        xps = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device="cuda")
        ws = single.workspace(k, B)
        single.ci_serve_group(xt, dt, hs, ps, ws, x_parity=xps, learned=learned)
        torch.cuda.synchronize()
        hs, ps, xps = hs.cpu().numpy(), ps.cpu().numpy(), xps.cpu().numpy()
        out = [np.load(tmp_path / f"r{r}_c{call}.npz") for r in range(world)]
        for r in range(k):   # main workers: h(x_r) for every group (the decoded slot aside)
            keep = drop != r
            assert relerr(out[r]["h"], ref["H"][:, r]) < TOL
            assert np.array_equal(out[r]["h"][keep], hs[keep, r])
        par = out[k]
        assert relerr(par["h"], ref["P"]) < TOL and np.array_equal(par["h"], ps)
        assert relerr(par["xp"].reshape(B, -1), ref["xp"].reshape(B, -1)) < TOL
        assert np.array_equal(par["xp"], xps)
        rows = B + Bp
        for p in range(world):   # decoded features of every rank's share of the groups
            b0, b1 = min(B, p * Bp), min(B, (p + 1) * Bp)
            for b in range(b0, b1):
                dec = out[p]["dec"][b - b0]
                if drop[b] < 0:
                    assert np.all(dec == 0)
                    continue
                assert relerr(dec, ref["R"][b, drop[b]]) < TOL
                assert np.array_equal(dec, hs[b, drop[b]])          # == single-GPU decode, bit for bit
                lo = 0
                for t, C in enumerate(heads):
                    lg = out[p]["logits"][lo:lo + rows * C].reshape(rows, C)[B + b - b0]
                    assert relerr(lg, ref["logits"][t][b, drop[b]]) < TOL
                    assert out[p]["labels"][t * rows + B + b - b0] == np.argmax(lg)
                    lo += rows * C
        for r in range(k):   # heads on each main worker's own result
            lo = 0
            for t, C in enumerate(heads):
                lg = out[r]["logits"][lo:lo + rows * C].reshape(rows, C)[:B]
                assert relerr(lg, ref["logits_n"][t][:, r]) < TOL
                lo += rows * C
