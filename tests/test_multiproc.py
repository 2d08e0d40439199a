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


# ------------------------------------------------------------------ C5 worker partition
class _OracleCompute:
    """CPU stand-in for GpuCompute (test only): per-rank compute from the f64 oracle."""

    def __init__(self, arch, params, k):
        self.arch, self.params, self.k, self.d = arch, params, k, arch.d

        class _M:
            pass
        self.model = _M()
        self.model.arch = arch

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float64)

    def forward_h(self, x):
        return torch.from_numpy(oracle.forward_h(self.arch, self.params, x.numpy(), nthreads=1))

    def inverse_h(self, h):
        return torch.from_numpy(oracle.inverse_h(self.arch, self.params, h.numpy(), nthreads=1))

    def encode_learned(self, x_all):
        return torch.from_numpy(oracle.encode_learned(self.arch, self.params, x_all.numpy(), nthreads=1))

    def coef(self, kind, worker, drop):
        d = torch.as_tensor(drop)
        if kind == 1:
            return torch.full((len(d),), (1.0 / self.k) if worker < self.k else 0.0, dtype=torch.float64)
        c = torch.where(d == worker, 0.0, -1.0).double() if worker < self.k else torch.full((len(d),), float(self.k),
                                                                                             dtype=torch.float64)
        return torch.where(d < 0, torch.zeros_like(c), c)

    def combine(self, f, coef):
        return f * coef[:, None]

    def classify(self, head, z):
        lg, lb = oracle.classify(self.arch, self.params, head, z.numpy())
        return torch.from_numpy(lg), torch.from_numpy(lb)


def _worker_c5(rank, world, port, B, learned, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_06445_b200.workers import serve_workers
    arch, k = fx.ARCH_TE, world - 1
    params = fx.make_weights(arch, 15)
    x = fx.make_inputs(arch, B, k, 5)
    drop = fx.make_drops(B, k, 105)
    drop[1] = -1                                  # one group without a loss
    comp = _OracleCompute(arch, params, k)
    xs = torch.from_numpy(x[:, rank].astype(np.float64)) if rank < k else None
    xa = torch.from_numpy(x.astype(np.float64)) if rank == k else None
    out = serve_workers(comp, dist, rank, world, k, torch.from_numpy(drop), x_slot=xs, x_all=xa, learned=learned)
    parts = [torch.empty_like(out["decoded"]) for _ in range(world)]
    dist.all_gather(parts, out["decoded"])
    if rank == 0:
        np.save(os.path.join(out_dir, "decoded.npy"), torch.cat(parts).numpy())
        np.save(os.path.join(out_dir, "logits_dec.npy"), out["logits_decoded"][1].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("learned", [False, True])
def test_worker_partition_gloo(tmp_path, learned):
    """C5 orchestration (k = 2 main workers + 1 parity worker, 3 ranks): the masked
    reduce-scatter decode equals the single-process oracle decode of the lost slot."""
    world, B = 3, 6
    mp.spawn(_worker_c5, args=(world, _free_port(), B, learned, str(tmp_path)), nprocs=world, join=True)
    arch, k = fx.ARCH_TE, world - 1
    params = fx.make_weights(arch, 15)
    x = fx.make_inputs(arch, B, k, 5)
    drop = fx.make_drops(B, k, 105)
    drop[1] = -1
    ref = oracle.serve_group(arch, params, x, drop, learned=learned, nthreads=1)
    dec = np.load(tmp_path / "decoded.npy")
    for b in range(B):
        if drop[b] < 0:
            assert np.all(dec[b] == 0)
        else:
            r = ref["R"][b, drop[b]]
            assert np.max(np.abs(dec[b] - r)) / np.max(np.abs(r)) < 1e-12
    lg = np.load(tmp_path / "logits_dec.npy")          # rank 0's partition, coarse head
    r0 = [b for b in range(B // world)]
    for b in r0:
        if drop[b] >= 0:
            assert np.max(np.abs(lg[b] - ref["logits"][1][b, drop[b]])) < 1e-10
