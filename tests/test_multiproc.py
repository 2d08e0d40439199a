"""World-size-2 CPU tests (gloo) of the multi-GPU host logic bench.py uses for N > 1:
group sharding (rank r serves global groups [r*B, (r+1)*B), no data-path collective),
counter-based input slices, and max-over-ranks timing.  Groups are independent units
(PAPER.md:211-214), so the sharded result must equal the single-process result bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fixtures as fx
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_input_slices_match_monolithic():
    arch = fx.ARCH_T
    full = fx.make_inputs(arch, 6, 2, 77)
    assert np.array_equal(fx.make_inputs_slice(arch, 2, 5, 2, 77), full[2:5])
    assert np.array_equal(fx.make_drops_slice(3, 9, 10, 5), fx.make_drops(9, 10, 5)[3:9])
    assert fx.shard(1, 4, 256) == (256, 512)


def _worker(rank, world, port, B, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = fx.CONFIGS["C1"]
    b0, b1 = fx.shard(rank, world, B)
    x = fx.make_inputs_slice(c.arch, b0, b1, c.k, c.seed_x)
    drop = fx.make_drops_slice(b0, b1, c.k, c.seed_drop)
    params = fx.make_weights(c.arch, c.seed_w)
    out = oracle.serve_group(c.arch, params, x, drop, nthreads=1)
    R = torch.from_numpy(out["R"])
    gathered = [torch.empty_like(R) for _ in range(world)]
    dist.all_gather(gathered, R)
    # max-over-ranks timing as bench.py does it
    t = torch.tensor([10.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(os.path.join(out_dir, "R.npy"), torch.cat(gathered).numpy())
        np.save(os.path.join(out_dir, "tmax.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_group_sharded_gloo_world2(tmp_path):
    world, B = 2, 3
    mp.spawn(_worker, args=(world, _free_port(), B, str(tmp_path)), nprocs=world, join=True)
    c = fx.CONFIGS["C1"]
    x = fx.make_inputs(c.arch, world * B, c.k, c.seed_x)
    drop = fx.make_drops(world * B, c.k, c.seed_drop)
    ref = oracle.serve_group(c.arch, fx.make_weights(c.arch, c.seed_w), x, drop, nthreads=1)
    assert np.array_equal(np.load(tmp_path / "R.npy"), ref["R"])
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 11.0
