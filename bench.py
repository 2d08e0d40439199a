#!/usr/bin/env python
"""Benchmark of the coded-inference hot path (BASELINE.json metric) on B200.

One step = one ci_serve_group call over B = 1024 coded groups of k = 10 CIFAR-shaped
queries (config C3): h on 10240 main queries, exact encode (mean + h^-1), h on the 1024
parity queries, decode of one random dropped worker per group, linear head + argmax.
The headline runs in the contract precision (CI_PREC_FP32: "f16x3" products -- both operands
split into fp16 hi + lo -- fp32 state and accumulators: <= 1e-3 vs the f64 oracle, checked in
the same run on 64 seeded groups); the bf16 and f16x2 (fp16-rounded weights) precisions are
reported beside it (`alt_precision`, with their own numerics vs the same oracle sample), as are
the MNIST-shaped C2 and the learned-encoder C4 workloads (`workloads`).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp32|f16x2|bf16] [--impl reference]

N > 1: one process per GPU.  Under torchrun the rank comes from the environment; when
`--gpus N` > 1 is given without a torchrun environment, bench.py re-launches itself under
`torch.distributed.run` with N processes (spawn_cmd).  Groups are sharded across ranks
(rank r serves global groups [r*1024, (r+1)*1024), no collective on the data path:
"scaling": "weak"); timing is a barrier + synchronize bracket, device-timed with CUDA events,
max over ranks (max_over_ranks).  Inputs rotate over 4 resident buffer sets (x + outputs
~1 GB > 126 MB L2).  The launcher / shard / max-timing helpers are exercised by
tests/test_multiproc.py with gloo at world size 2.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

# one hardware queue per CUDA stream (first-k harness: k + 2 + in-flight streams; must be set
# before the CUDA context exists)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fixtures as fx  # noqa: E402

METRIC = "coded query groups/sec (k=10, CIFAR-shape) at 1/2/4/8 B200; % tensor/HBM peak"
UNIT = "groups/s"
NBUF = 4
TOL = 1e-3          # north star: max relative error on fp32 features and logits
DTYPE = {"fp32": "f16x3", "f16x2": "f16x2", "bf16": "bf16"}   # arithmetic of the tensor-core products
MMAS = {"fp32": 3, "f16x2": 2, "bf16": 1}                       # MMAs issued per algorithmic product


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- launcher
def dist_env():
    """(rank, world, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_cmd(argv, nproc, port):
    """The torchrun command that runs this script with one process per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def maybe_spawn(args, argv):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run; returns the exit
    code, or None when this process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    return subprocess.call(spawn_cmd(argv, args.gpus, free_port()))


def max_over_ranks(ms, dist, device=None):
    """Slowest rank's device time (all_reduce MAX); identity for one process."""
    if dist is None:
        return float(ms)
    import torch
    t = torch.tensor([float(ms)], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50",
                                          "-i", str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power)}


# ----------------------------------------------------------------------------- numerics
def relerr(a, ref):
    """max over samples of ||a_s - r_s||_inf / ||r_s||_inf."""
    a = np.asarray(a, np.float64).reshape(-1, np.shape(ref)[-1])
    r = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


def sample_groups(B, S, seed=2106):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(B, min(S, B), replace=False))


def numerics(cfg, precision, groups, drop, out, ref):
    """GPU outputs of the sampled groups vs the f64 oracle's (same inputs and weights)."""
    arch, k = cfg.arch, cfg.k
    S = len(groups)
    bi = np.arange(S)
    R, P, XP = out["R"][groups], out["P"][groups], out["xp"][groups]
    dg = drop[groups]
    e = {"groups_checked": int(S), "precision": precision, "dtype": DTYPE[precision],
         "max_rel_err_features": relerr(R, ref["R"]),
         "max_rel_err_decoded": relerr(R[bi, dg], ref["R"][bi, dg]),
         "max_rel_err_parity": relerr(P, ref["P"]),
         "max_rel_err_parity_input": relerr(XP.reshape(S, -1), ref["xp"].reshape(S, -1))}
    n = cfg.B * k
    lo = 0
    agree, agree_dec, worst_logit = [], [], 0.0
    for t, C in enumerate(arch.heads):
        L = out["logits"][lo:lo + n * C].reshape(cfg.B, k, C)[groups]
        lab = out["labels"][t * n:(t + 1) * n].reshape(cfg.B, k)[groups]
        worst_logit = max(worst_logit, relerr(L, ref["logits"][t]))
        agree.append(float(np.mean(lab == ref["labels"][t])))
        agree_dec.append(float(np.mean(lab[bi, dg] == ref["labels"][t][bi, dg])))
        lo += n * C
    e["max_rel_err_logits"] = worst_logit
    e["label_agreement"] = min(agree) if agree else None
    e["label_agreement_decoded"] = min(agree_dec) if agree_dec else None
    worst = max(e["max_rel_err_features"], e["max_rel_err_parity"], e["max_rel_err_parity_input"],
                e["max_rel_err_logits"])
    e["tolerance"] = TOL
    e["pass"] = bool(worst <= TOL)
    if precision != "fp32":
        e["note"] = (f"{DTYPE[precision]} products: bound and label agreement reported, not promised <= 1e-3 "
                     f"(north star; only CI_PREC_FP32 is the contract precision)")
    return e


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the f64 CPU oracle as it stands, on a bounded sample per step."""
    import oracle
    if rank != 0:
        return
    cfg = fx.CONFIGS[args.config]
    params = fx.make_weights(cfg.arch, cfg.seed_w)
    S = args.ref_groups
    x = fx.make_inputs(cfg.arch, S, cfg.k, cfg.seed_x)
    drop = fx.make_drops(S, cfg.k, cfg.seed_drop)
    oracle.build()
    learned = bool(cfg.arch.encoder)
    for _ in range(args.warmup):
        oracle.serve_group(cfg.arch, params, x, drop, learned=learned, fp_iters=cfg.arch.fp_iters)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.serve_group(cfg.arch, params, x, drop, learned=learned, fp_iters=cfg.arch.fp_iters)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = S * args.steps / total
    cores = os.cpu_count()
    sample = f"{S} groups of {cfg.name} (k={cfg.k}) per step, f64 oracle, {cores} threads"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "k": cfg.k, "groups_per_step": S,
                                            "arch": fx.arch_summary(cfg.arch)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- C5
def run_c5(args, rank, world, local):
    """Config C5: k = 7 main workers + 1 parity worker, one per GPU (8 ranks), 1024 groups per
    step, through ci_serve_group with a CI_SHARD_WORKERS communicator: encode exact (X2: the
    parity GPU reads the mains' features over NVLink and forms the mean, then h^-1 and h) or
    learned (encoder on the parity GPU); decode = K11, every GPU reading its share of the groups
    from all peers' windows.  Drops are masked, not waited on (PAPER.md:669's straggler delay is
    the first_k harness)."""
    cfg = fx.CONFIGS["C5"]
    k, B = cfg.k, cfg.B
    if world != k + 1:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "config": {"workload": "C5"},
                              "unavailable": f"C5 needs {k + 1} ranks (one per worker), got {world}"}))
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_2106_06445_b200 import codedinv as ci
    from paper_2106_06445_b200.workers import WorkerBuffers, make_comm, serve_worker
    arch = cfg.arch
    learned = args.encode == "learned"
    model = ci.Model(arch, fx.make_weights(arch, cfg.seed_w), args.precision, device=local)
    comm = make_comm(dist, ci.CI_SHARD_WORKERS, B, model.d, device=local)
    bufs = WorkerBuffers(model, k, B, torch.device("cuda", local))
    dev = torch.device("cuda", local)
    x = fx.make_inputs(arch, B, k, cfg.seed_x)
    drop = torch.from_numpy(fx.make_drops(B, k, cfg.seed_drop)).to(dev)
    if rank < k:
        xin = torch.from_numpy(np.ascontiguousarray(x[:, rank])).to(dev)
    else:
        xin = torch.from_numpy(x).to(dev) if learned else None
    step = lambda: serve_worker(model, comm, xin, drop, bufs, learned=learned)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1), dist)
    model.ci_check(bufs.ws)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": B * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "none (fixed 8-worker partition)",
                          "vs_baseline": None, "dtype": DTYPE[args.precision], "data": "synthetic",
                          "config": {"workload": "C5", "k": k, "groups_per_step": B, "encode": args.encode,
                                     "parallelism": "worker-per-GPU (k=7 main + 1 parity); mean and decode "
                                                    "fused over peer memory (NVLink)"}}), flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- our path
class Workload:
    """Resident device buffers of one config: NBUF rotating input / output sets (this rank's
    groups of each global workload: counter-based slices, no rank generates others' groups)."""

    def __init__(self, cfg, rank, world, dev, nbuf=NBUF):
        import torch
        self.cfg, self.dev = cfg, dev
        arch, k, B = cfg.arch, cfg.k, cfg.B
        self.b0, self.b1 = fx.shard(rank, world, B)
        self.params = fx.make_weights(arch, cfg.seed_w)
        self.x_host0 = fx.make_inputs_slice(arch, self.b0, self.b1, k, cfg.seed_x)
        self.drop_host0 = fx.make_drops_slice(self.b0, self.b1, k, cfg.seed_drop)
        self.xs = [torch.from_numpy(self.x_host0 if i == 0 else
                                    fx.make_inputs_slice(arch, self.b0, self.b1, k, cfg.seed_x + 7919 * i)).to(dev)
                   for i in range(nbuf)]
        self.drops = [torch.from_numpy(self.drop_host0 if i == 0 else
                                       fx.make_drops_slice(self.b0, self.b1, k, cfg.seed_drop + 7919 * i)).to(dev)
                      for i in range(nbuf)]
        d = arch.d
        self.ncls = sum(arch.heads)
        self.hs = [torch.empty(B, k, d, device=dev) for _ in range(nbuf)]
        self.ps = [torch.empty(B, d, device=dev) for _ in range(nbuf)]
        self.xps = [torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device=dev) for _ in range(nbuf)]
        self.lg = [torch.empty(max(B * k * self.ncls, 1), device=dev) for _ in range(nbuf)]
        self.lb = [torch.empty(max(B * k * len(arch.heads), 1), dtype=torch.int32, device=dev) for _ in range(nbuf)]
        self.learned = bool(arch.encoder)
        self.nbuf = nbuf

    def serve(self, model, ws, j, stream=None):
        model.ci_serve_group(self.xs[j], self.drops[j], self.hs[j], self.ps[j], ws, x_parity=self.xps[j],
                             logits=self.lg[j], labels=self.lb[j], learned=self.learned, stream=stream)

    def outputs(self, j=0):
        return dict(R=self.hs[j].cpu().numpy(), P=self.ps[j].cpu().numpy(), xp=self.xps[j].cpu().numpy(),
                    logits=self.lg[j].cpu().numpy(), labels=self.lb[j].cpu().numpy())


def timed_run(ci, wl, model, steps, warmup, nin, dist=None, measure=True, prof=False, graph=False, local=0):
    """W warm-up steps, then EXACTLY `steps` steps bracketed by barrier + synchronize, device-
    timed with CUDA events on the launching stream; nin request batches in flight alternate over
    nin streams (own workspaces).  graph: replay a CUDA graph of one serve call (nin = 1)."""
    import torch
    k, B = wl.cfg.k, wl.cfg.B
    stream = torch.cuda.current_stream()
    wss = [model.workspace(k, B) for _ in range(nin)]
    streams = [stream] + [torch.cuda.Stream(device=wl.dev) for _ in range(nin - 1)]
    graphs = None
    if graph:
        assert nin == 1
        wl.serve(model, wss[0], 0)
        torch.cuda.synchronize()
        ci.ci_test_launch_count(reset=True)
        graphs = []
        for j in range(wl.nbuf):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                wl.serve(model, wss[0], j)
            graphs.append(g)
        torch.cuda.synchronize()
        per_call = ci.ci_test_launch_count(reset=True) / wl.nbuf

    def step(i):
        j = i % wl.nbuf
        if graphs is not None:
            graphs[j].replay()
            return
        wl.serve(model, wss[i % nin], j, stream=streams[i % nin])

    for s_ in streams[1:]:
        s_.wait_stream(stream)
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    ci.ci_test_prof_read()
    ci.ci_test_launch_count(reset=True)
    sampler = ClockSampler(local)
    if measure:
        sampler.start()
        time.sleep(0.2)
    ci.ci_test_prof_enable(prof and nin == 1 and not graph)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s_ in streams[1:]:
        s_.wait_stream(stream)
    for i in range(steps):
        step(i)
    for s_ in streams[1:]:
        stream.wait_stream(s_)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ci.ci_test_prof_enable(False)
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop() if measure else None
    launches = ci.ci_test_launch_count(reset=True)
    if graphs is not None:
        launches = int(round(per_call * steps))
    kms, kl, kfl = ci.ci_test_prof_read()
    for w_ in wss:
        model.ci_check(w_)
    ms = max_over_ranks(ms, dist, wl.dev)
    return dict(ms=ms, clocks=clocks, launches=launches, kms=kms, klaunch=kl, kflops=kfl, ws=wss[0])


def stage_kernel_names(ci, arch, precision):
    """The kernel each stage of h runs on (planner query: TS kernels / interleaved raster / k_stage)."""
    pm = {"bf16": 0, "f16x2": 1, "fp32": 2}[precision]
    names = []
    for (C, H, W, c, m, nb) in arch.stage_shapes():
        q = -c if arch.block == "residual" else c
        try:
            p = ci.ci_test_plan(H, W, q, m, pm)
        except Exception:
            names.append("k_stage")
            continue
        names.append({1: "k_stage_ts", 2: "k_stage_ts2"}.get(p.get("ts", 0), "k_stage") +
                     (" (interleaved raster)" if p.get("nopad") == 2 else ""))
    return names


def stage_roofline(run, peaks, peak_src, precision, step_ms, measured_in, names=None):
    """Roofline of the dominant kernels (the fused tcgen05 stage kernels of h, summed) from live
    CUDA events."""
    kms, kfl, kl = run["kms"], run["kflops"], run["klaunch"]
    stage_ms, stage_fl = sum(kms), sum(kfl)
    if stage_ms <= 0:
        return None, {}
    achieved = stage_fl / (stage_ms / 1e3) / 1e12
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"k_stage_{precision}")
        except Exception:
            traffic = None
    mult = MMAS[precision]
    label = " + ".join(dict.fromkeys(n.split(" (")[0] for n in names)) if names else "k_stage"
    roof = {"bound": "tensor", "kernel": f"fused tcgen05 stage kernels of h ({label}), summed",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_source": f"{peak_src} bf16_tflops_sustained (dense bf16 cuBLAS, 4 s loop); fp16 runs at the "
                           f"same kind::f16 rate",
            "frac_of_burst": achieved / peaks["bf16_tflops"],
            "issued_mma_multiplier": mult, "issued_frac": achieved * mult / peak,
            "traffic": traffic, "share_of_step": stage_ms / step_ms, "measured_in": measured_in,
            "algorithmic_flops": "n * blocks * 36 * H * W * c * m per launch (2 per MAC of both 3x3 convs)"}
    kernels = {}
    for s in range(4):
        if kl[s]:
            kernels[f"k_stage[s{s}]"] = {"kernel": names[s] if names and s < len(names) else "k_stage",
                                         "launches": kl[s], "ms_per_launch": kms[s] / kl[s],
                                         "tflops": kfl[s] / (kms[s] / 1e3) / 1e12,
                                         "frac_of_peak": kfl[s] / (kms[s] / 1e3) / 1e12 / peak}
    return roof, kernels


def measure_workload(ci, wl, precision, args, dist, local, peaks, peak_src, nin, graph=False, measure=True,
                     reps=0):
    """Throughput (+ reps) and the single-stream roofline pass of one workload / precision."""
    model = ci.Model(wl.cfg.arch, wl.params, precision, device=local)
    run = timed_run(ci, wl, model, args.steps, args.warmup, nin, dist=dist, measure=measure, graph=graph,
                    local=local)
    world = dist.get_world_size() if dist else 1
    B = wl.cfg.B
    res = {"precision": precision, "dtype": DTYPE[precision], "value": world * B * args.steps / (run["ms"] / 1e3),
           "ms_per_step": run["ms"] / args.steps, "clocks": run["clocks"], "gpu_launches": run["launches"],
           "inflight": nin, "cuda_graph": graph}
    if reps:
        vals = [world * B * args.steps / (timed_run(ci, wl, model, args.steps, 1, nin, dist=dist, measure=False,
                                                    graph=graph, local=local)["ms"] / 1e3) for _ in range(reps)]
        res["reps"] = {"n": reps, "median": float(np.median(vals)), "p10": float(np.percentile(vals, 10)),
                       "p90": float(np.percentile(vals, 90)), "steps_per_rep": args.steps}
    prof = timed_run(ci, wl, model, max(3, args.steps // 2), 3, 1, dist=dist, measure=False, prof=True, local=local)
    res["roofline"], res["kernels"] = stage_roofline(prof, peaks, peak_src, precision, prof["ms"],
                                                     "single-stream pass" if nin > 1 or graph else "timed region",
                                                     names=stage_kernel_names(ci, wl.cfg.arch, precision))
    res["model"], res["ws"] = model, run["ws"]
    return res


def hbm_extras(ci, dev, stream, peaks, k, d):
    """Encode-mean / decode standalone against HBM (L2-cold, 1.1 GB) and the online decoding
    completion event (f2) vs the batch decode."""
    import torch
    hbm = {}
    Bd = 8192
    Hb = torch.empty(Bd, k, d, device=dev).uniform_()
    Pb = torch.empty(Bd, d, device=dev).uniform_()
    Db = torch.empty(Bd, dtype=torch.int32, device=dev)
    ci.ci_make_drops(k, Bd, 99, Db)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
    ws0 = torch.zeros(256, dtype=torch.uint8, device=dev)
    Mb = torch.empty(Bd, d, device=dev)
    for name in ("decode", "mean"):
        tms = []
        for it in range(6):
            flush.zero_()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            if name == "decode":
                ci.ci_decode(Hb, Pb, Db, ws0)
            else:
                ci.ci_test_mean(Hb, Mb)
            b_.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                tms.append(a_.elapsed_time(b_))
        t = float(np.median(tms))
        byts = Bd * ((k + 1) * d * 4 + 4) if name == "decode" else Bd * (k + 1) * d * 4
        hbm[name] = {"groups": Bd, "ms": t, "bytes": byts, "achieved": byts / (t / 1e3) / 1e9,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": byts / (t / 1e3) / 1e9 / peaks["hbm_gbs"],
                     "note": "L2 flushed (256 MB write) before each launch"}
    del Hb, Pb, Mb
    online = {}

    def t_of(fn, setup=None):
        ts = []
        for it in range(5):
            flush.zero_()
            if setup:
                setup()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            fn()
            b_.record(stream)
            torch.cuda.synchronize()
            if it >= 1:
                ts.append(a_.elapsed_time(b_))
        return float(np.median(ts)) * 1e3

    for kk in (2, 4, 10, 30):
        Bo = 1024
        est = torch.zeros(Bo, kk, d, device=dev)
        val = torch.randn(Bo, d, device=dev)
        Hk = torch.randn(Bo, kk, d, device=dev)
        Dk = torch.zeros(Bo, dtype=torch.int32, device=dev)
        rec = ((1 << kk) - 1) & ~1          # mains 1..k-1 in, main 0 missing, parity pending
        state0 = torch.full((Bo,), (rec << 32) | rec, dtype=torch.int64, device=dev)
        st_ = state0.clone()
        task = torch.full((Bo,), kk, dtype=torch.int32, device=dev)
        wso = torch.zeros(256, dtype=torch.uint8, device=dev)
        online[f"k={kk}"] = {
            "completing_event_us": t_of(lambda: ci.ci_online_update(kk, est, st_, task, val, wso),
                                        setup=lambda: st_.copy_(state0)),
            "batch_decode_us": t_of(lambda: ci.ci_decode(Hk, val, Dk, wso))}
    hbm["online_decode"] = {"groups": 1024, "per_k": online,
                            "note": "completing event = the parity arrives after k-1 mains: one fma "
                                    "per element of the missing estimate; batch = k P - sum of k-1 mains"}
    return hbm


def nearest_rank(v, p):
    """Nearest-rank percentile (SPEC.md LatencyStats): sorted[ceil(p/100 * N) - 1]."""
    v = np.sort(np.asarray(v))
    return float(v[max(0, int(np.ceil(p / 100.0 * len(v))) - 1)])


def first_k_extras(ci, dev, precision, queries=1000, delay_ns=100_000_000, inflight=16):
    """f2: first-k gated serving with online decoding (ci_serve_first_k) on the learned-encoder
    arch (the parity worker encodes from the raw queries), one group of k = 10
    CIFAR-shaped queries per query, 0.1 s injected on one random main worker per query
    (PAPER.md:669).  Three arms (SPEC.md latency_comparison): coded with the straggler, uncoded
    (waits for all k) with the straggler, coded without stragglers; plus the completing event's
    online-update cost vs k (App. C: independent of k)."""
    import torch
    cfg = fx.CONFIGS["C4"]
    arch = cfg.arch
    model = ci.Model(arch, fx.make_weights(arch, cfg.seed_w), precision)

    def arm(k, Q, strag, uncoded, inflight=inflight):
        x = torch.from_numpy(fx.make_inputs(arch, Q, k, cfg.seed_x + k)).to(dev)
        feats = torch.empty(Q, k, arch.d, device=dev)
        lg = torch.empty(Q * k * sum(arch.heads), device=dev)
        lb = torch.empty(Q * k * len(arch.heads), dtype=torch.int32, device=dev)
        rec = torch.zeros(Q, 4, dtype=torch.int64, device=dev)
        ws = model.workspace_first_k(k, inflight)
        model.ci_serve_first_k(x, strag[:8], delay_ns, feats[:8], lg, lb, rec, ws, max_inflight=inflight,
                               uncoded=uncoded)   # warm-up (8 queries)
        t0 = time.perf_counter()
        model.ci_serve_first_k(x, strag, delay_ns, feats, lg, lb, rec, ws, max_inflight=inflight, uncoded=uncoded)
        wall = time.perf_counter() - t0
        r = rec.cpu().numpy()
        lat = r[:, 0] / 1e6
        return {"queries": Q, "p50_ms": nearest_rank(lat, 50), "p99_ms": nearest_rank(lat, 99),
                "p999_ms": nearest_rank(lat, 99.9), "mean_ms": float(lat.mean()),
                "update_us_median": float(np.median(r[:, 1]) / 1e3), "heads_us_median": float(np.median(r[:, 2]) / 1e3),
                "degraded_frac": float(np.mean(r[:, 3] >> 32)), "wall_s": wall}

    k = cfg.k
    rng = np.random.default_rng(669)
    strag = rng.integers(0, k, queries).astype(np.int32)
    none = np.full(queries, -1, np.int32)
    out = {"k": k, "delay_ms": delay_ns / 1e6, "inflight": inflight, "precision": precision,
           "coded_straggler": arm(k, queries, strag, False),
           "uncoded_straggler": arm(k, max(queries // 3, 64), strag, True),
           "coded_no_straggler": arm(k, queries, none, False, inflight=1)}
    per_k = {}
    for kk in (2, 4, 10):
        a = arm(kk, 200, np.full(200, -1, np.int32), False, inflight=1)
        per_k[f"k={kk}"] = {"update_us_median": a["update_us_median"], "heads_us_median": a["heads_us_median"],
                            "p50_ms": a["p50_ms"]}
    out["completing_event_vs_k"] = per_k
    out["note"] = ("latency = device globaltimer from query submission to the heads' output on the k recovered "
                   "features; workers = CUDA streams of one GPU; update = the completing event's online "
                   "update (App. C), heads = the linear heads on the k features; straggler arms keep up to "
                   "`inflight` queries in flight (a slot frees when its straggler reports), the no-straggler "
                   "and per-k arms run one query at a time (no queueing)")
    return out


def e2e_measure(ci, wl, model, args, dist, nin):
    """Same metric through the host-buffer C-ABI call: pinned H2D of x + drop and D2H of every
    output inside the device-timed region."""
    import torch
    arch, k, B = wl.cfg.arch, wl.cfg.k, wl.cfg.B
    d, ncls = arch.d, wl.ncls
    stream = torch.cuda.current_stream()
    xh = torch.from_numpy(wl.x_host0).pin_memory()
    dh = torch.from_numpy(wl.drop_host0).pin_memory()
    sets = []
    for _ in range(nin):
        hh = torch.empty(B, k, d).pin_memory()
        ph = torch.empty(B, d).pin_memory()
        lgh = torch.empty(max(B * k * ncls, 1)).pin_memory()
        lbh = torch.empty(max(B * k * len(arch.heads), 1), dtype=torch.int32).pin_memory()
        sets.append(((xh.numpy(), dh.numpy(), hh.numpy(), ph.numpy(), lgh.numpy(), lbh.numpy()),
                     model.workspace(k, B, host=True)))
    estreams = [stream] + [torch.cuda.Stream(device=wl.dev) for _ in range(nin - 1)]

    def e2e_call(i):
        a_h, w_h = sets[i % nin]
        model.ci_serve_group_host(*a_h, w_h, learned=wl.learned, stream=estreams[i % nin], sync=(nin == 1))

    for i in range(2 * nin):
        e2e_call(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e_steps = max(3, args.steps)   # as many steps as the device-timed line: same pipeline fill / drain share
    e_steps += (-e_steps) % nin
    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_.record(stream)
    for s_ in estreams[1:]:
        s_.wait_stream(stream)
    for i in range(e_steps):
        e2e_call(i)
    for s_ in estreams[1:]:
        stream.wait_stream(s_)
    b_.record(stream)
    torch.cuda.synchronize()
    for _, w_h in sets:
        model.ci_check(w_h)
    ems = max_over_ranks(a_.elapsed_time(b_), dist, wl.dev)
    world = dist.get_world_size() if dist else 1
    hh, ph, lgh, lbh = (torch.from_numpy(a) for a in sets[0][0][2:])
    return {"value": world * B * e_steps / (ems / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(xh.numel() * 4 + dh.numel() * 4),
            "d2h_bytes_per_step": int(hh.numel() * 4 + ph.numel() * 4 + lgh.numel() * 4 + lbh.numel() * 4),
            "steps": e_steps, "inflight": nin,
            "note": "ci_serve_group_host(_async): pinned H2D of x+drop, D2H of h_out, h_parity, logits, "
                    "labels inside the device-timed region; calls alternate over `inflight` streams"}


def oracle_reference(cfg, wl, groups):
    """f64 oracle on the sampled groups of buffer 0 (the checker; timed = cpu_baseline)."""
    import oracle
    t0 = time.perf_counter()
    ref = oracle.serve_group(cfg.arch, wl.params, wl.x_host0[groups], wl.drop_host0[groups],
                             learned=bool(cfg.arch.encoder), fp_iters=cfg.arch.fp_iters)
    return ref, time.perf_counter() - t0


def checked(ci, wl, res, groups, ref):
    """Re-run buffer 0 with the measured model and compare the sampled groups with the oracle."""
    import torch
    wl.serve(res["model"], res["ws"], 0)
    torch.cuda.synchronize()
    res["model"].ci_check(res["ws"])
    return numerics(wl.cfg, res["precision"], groups, wl.drop_host0, wl.outputs(0), ref)


def public(res):
    return {k_: v for k_, v in res.items() if k_ not in ("model", "ws")}


def encoder_overhead(ci, wl, model, dev, stream):
    """Learned-encoder time / time of h on the k main queries, 1024 groups, k in {2, 4, 10}
    (Figs. 6-7 analogue)."""
    import torch
    arch, B = wl.cfg.arch, wl.cfg.B
    out = {}
    for kk in (2, 4, 10):
        xk = torch.from_numpy(fx.make_inputs_slice(arch, 0, B, kk, wl.cfg.seed_x)).to(dev)
        wsk = model.workspace(kk, B)
        hk = torch.empty(B * kk, arch.d, device=dev)
        xpk = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device=dev)

        def timed(fn, reps=5):
            fn()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(reps):
                fn()
            b_.record(stream)
            torch.cuda.synchronize()
            return a_.elapsed_time(b_) / reps
        t_enc = timed(lambda: model.ci_encode(None, xpk, wsk, x=xk, learned=True))
        t_h = timed(lambda: model.ci_forward_h(xk.reshape(B * kk, arch.in_c, arch.in_h, arch.in_w), hk, wsk))
        out[str(kk)] = {"encoder_ms": t_enc, "h_ms": t_h, "overhead": t_enc / t_h}
        del xk, wsk, hk, xpk
    return out


def main():
    argv = sys.argv[1:]
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "f16x2", "bf16"])
    ap.add_argument("--config", default="C3", choices=["C3", "C4", "C5", "C2", "C1", "C3R"])
    ap.add_argument("--encode", default="exact", choices=["exact", "learned"], help="C5 parity encode mode")
    ap.add_argument("--ref-groups", type=int, default=8, help="oracle sample groups per step (--impl reference)")
    ap.add_argument("--cpu-groups", type=int, default=64, help="oracle sample: numerics + cpu_baseline")
    ap.add_argument("--reps", type=int, default=5, help="extra timed repetitions (median / p10 / p90)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other-precision line items")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the standalone HBM / online-decode / label-generation / other-workload items")
    ap.add_argument("--inflight", type=int, default=2, choices=[1, 2, 3, 4],
                    help="request batches in flight (2: consecutive steps alternate between two CUDA streams)")
    args = ap.parse_args(argv)
    assert args.warmup >= 1 and args.steps >= 1

    rc = maybe_spawn(args, argv)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.config == "C5":
        return run_c5(args, rank, world, local)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}")
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2106_06445_b200 import codedinv as ci

    cfg = fx.CONFIGS[args.config]
    arch, k, B = cfg.arch, cfg.k, cfg.B
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    peaks, peak_src = load_peaks()
    wl = Workload(cfg, rank, world, dev)

    # --- headline: the contract precision, 2 request batches in flight
    main_res = measure_workload(ci, wl, args.precision, args, dist, local, peaks, peak_src, args.inflight,
                                reps=args.reps)
    extras = rank == 0 and world == 1 and not args.no_extras

    hbm = hbm_extras(ci, dev, stream, peaks, k, arch.d) if extras else {}
    first_k = first_k_extras(ci, dev, args.precision) if extras else None
    e2e = None if args.no_e2e else e2e_measure(ci, wl, main_res["model"], args, dist, args.inflight)

    # --- bulk encoder-label generation (f4): h on the k inputs + mean + h^-1
    label_gen = None
    if extras and not wl.learned:
        model, wsl = main_res["model"], main_res["ws"]
        hl = torch.empty(B, k, arch.d, device=dev)
        xl = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device=dev)

        def gen(j):
            model.ci_forward_h(wl.xs[j].view(B * k, arch.in_c, arch.in_h, arch.in_w), hl.view(B * k, arch.d), wsl)
            model.ci_encode(hl, xl, wsl)
        for j in range(3):
            gen(j % NBUF)
        torch.cuda.synchronize()
        reps = 8
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        for j in range(reps):
            gen(j % NBUF)
        b_.record(stream)
        torch.cuda.synchronize()
        lms = a_.elapsed_time(b_) / reps
        label_gen = {"pairs_per_s": B / (lms / 1e3), "ms_per_1024": lms * 1024 / B,
                     "seconds_for_50000": 50000 / (B / (lms / 1e3)), "precision": args.precision,
                     "note": "exact (x-tuple, h^-1(mean h)) training pairs for the learned encoder"}
        del hl, xl

    # --- oracle on a bounded sample: numerics of every measured precision + cpu_baseline
    cpu, num, ref = None, None, None
    groups = sample_groups(B, args.cpu_groups)
    if rank == 0 and not args.no_cpu_baseline:
        ref, dt = oracle_reference(cfg, wl, groups)
        cpu = {"value": len(groups) / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{len(groups)} seeded groups of {cfg.name} (k={k}: {len(groups) * (k + 2)} h-equivalents, "
                         f"f64 C oracle, pthreads over images), wall {dt:.1f} s"}
        num = checked(ci, wl, main_res, groups, ref)

    # --- other precisions, same workload: throughput + roofline + numerics vs the same oracle
    alt = None
    if not args.no_alt:
        alt = {}
        for other in [p_ for p_ in ("bf16", "f16x2", "fp32") if p_ != args.precision]:
            r2 = measure_workload(ci, wl, other, args, dist, local, peaks, peak_src, args.inflight, measure=False)
            if ref is not None:
                r2["numerics"] = checked(ci, wl, r2, groups, ref)
            alt[other] = public(r2)
            alt[other].pop("clocks", None)
            del r2

    # --- the other BASELINE workloads at the headline precision: C2 (MNIST-shaped, launch-bound:
    #     CUDA graph of the serve call) and C4 (learned encoder, heads 10 + 2)
    workloads = {}
    enc_over = None
    if extras:
        for name, graph, S in (("C2", True, 256), ("C4", False, args.cpu_groups)):
            cw = fx.CONFIGS[name]
            w2 = Workload(cw, 0, 1, dev)
            r = measure_workload(ci, w2, args.precision, args, None, local, peaks, peak_src,
                                 1 if graph else args.inflight, graph=graph, measure=False)
            if not args.no_cpu_baseline:
                g2 = sample_groups(cw.B, S, seed=2107)
                ref2, dt2 = oracle_reference(cw, w2, g2)
                r["numerics"] = checked(ci, w2, r, g2, ref2)
                r["cpu_baseline"] = {"value": len(g2) / dt2, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                                     "sample": f"{len(g2)} groups of {name}, wall {dt2:.1f} s"}
            if name == "C4":
                enc_over = encoder_overhead(ci, w2, r["model"], dev, stream)
            r["config"] = {"workload": name, "k": cw.k, "groups_per_gpu": cw.B, "arch": fx.arch_summary(cw.arch),
                           "image": f"{cw.arch.in_c}x{cw.arch.in_h}x{cw.arch.in_w}",
                           "encode": "learned encoder (Arch E), heads 10 + 2" if cw.arch.encoder else
                           "exact h^-1(mean h)"}
            workloads[name] = public(r)
            workloads[name].pop("clocks", None)
            del w2, r

    if rank == 0:
        line = {"metric": METRIC, "value": main_res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[args.precision],
                "data": "synthetic",
                "config": {"workload": cfg.name, "k": k, "groups_per_gpu": B, "global_groups": B * world,
                           "queries_per_group": k + 1,
                           "image": f"{arch.in_c}x{arch.in_h}x{arch.in_w}",
                           "arch": fx.arch_summary(arch),
                           "encode": "learned encoder (Arch E)" if wl.learned else "exact h^-1(mean h)",
                           "precision": args.precision,
                           "parallelism": f"group-sharded x{world}",
                           "l2": f"inputs rotate over {NBUF} resident buffer sets (x+outputs ~1 GB > L2)",
                           "inflight": args.inflight},
                "roofline": main_res["roofline"], "kernels": main_res["kernels"],
                "reps": main_res.get("reps"), "hbm": hbm,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": main_res["gpu_launches"], "clocks": main_res["clocks"],
                "numerics": num, "alt_precision": alt, "workloads": workloads}
        if enc_over is not None:
            line["encoder_overhead"] = enc_over
        if label_gen:
            line["label_generation"] = label_gen
        if first_k:
            line["first_k"] = first_k
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
