"""Multi-process CPU tests of the host logic of the multi-GPU paths.

Group-sharded data parallelism (bench.py for N > 1; gloo, world size 2): rank r serves global
groups [r*B, (r+1)*B) with no data-path collective, counter-based input slices, bench.py's own
rank discovery / max-over-ranks timing / self-spawn.  Groups are independent units
(PAPER.md:211-214), so the sharded result equals the single-process result bit-exactly.
Worker partition (C5): the node-local rendezvous that bootstraps ci_comm_create."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import fixtures as fx
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_bench_spawns_n_ranks_itself():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (spawn_cmd); the
    reference arm runs on CPU, so the whole launcher path executes here: rank 0 prints one JSON
    line with n_gpus = 2, rank 1 exits 0."""
    import json
    import subprocess
    import sys
    env = {k_: v for k_, v in os.environ.items() if k_ not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, bench.__file__, "--impl", "reference", "--gpus", "2", "--config", "C1",
                          "--steps", "1", "--warmup", "1", "--ref-groups", "1"], capture_output=True, text=True,
                         env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    cmd = bench.spawn_cmd(["--gpus", "4"], 4, 29500)
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd


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
    # bench.py's own rank discovery and max-over-ranks timing
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    assert bench.dist_env() == (rank, world, rank)
    t = np.array([bench.max_over_ranks(10.0 + rank, dist)])
    if rank == 0:
        np.save(os.path.join(out_dir, "R.npy"), torch.cat(gathered).numpy())
        np.save(os.path.join(out_dir, "tmax.npy"), t)
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


# ------------------------------------------------------------------ C5 communicator bootstrap
def _rendezvous_worker(rank, world, uid, out_dir):
    from paper_2106_06445_b200 import codedinv as ci
    got = ci.ci_test_rendezvous(uid, world, rank, bytes([rank + 1]) * 40)
    np.save(os.path.join(out_dir, f"rv{rank}.npy"), np.frombuffer(b"".join(got), np.uint8))


def test_comm_rendezvous_world4(tmp_path):
    """The host rendezvous of ci_comm_create (POSIX shared memory named by ci_comm_unique_id):
    4 processes each publish 40 bytes and all receive every rank's payload in rank order."""
    from paper_2106_06445_b200 import build
    build.build()
    from paper_2106_06445_b200 import codedinv as ci
    uid = ci.ci_comm_unique_id()
    assert len(uid) == ci.CI_COMM_ID_BYTES and any(uid[:16]) and ci.ci_comm_unique_id() != uid
    world = 4
    mp.spawn(_rendezvous_worker, args=(world, uid, str(tmp_path)), nprocs=world, join=True)
    want = np.frombuffer(b"".join(bytes([q + 1]) * 40 for q in range(world)), np.uint8)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"rv{r}.npy"), want)
    assert not os.path.exists("/dev/shm/codedinv_" + uid[:16].hex())   # the name is unlinked after use
