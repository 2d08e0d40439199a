#!/usr/bin/env python
"""Benchmark of the coded-inference hot path (BASELINE.json metric) on B200.

One step = one ci_serve_group call over B = 1024 coded groups of k = 10 CIFAR-shaped
queries (config C3): h on 10240 main queries, exact encode (mean + h^-1), h on the 1024
parity queries, decode of one random dropped worker per group, linear head + argmax.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision bf16|fp32] [--impl reference]

N > 1: launched by torchrun, one process per GPU; groups are sharded across ranks (each
rank serves its own 1024 groups, no collective on the data path: "scaling": "weak");
timing is a barrier + synchronize bracket, device-timed with CUDA events, max over ranks.
Inputs rotate over 4 resident buffer sets (x + outputs ~1 GB > 126 MB L2).
Rank r serves global groups [r*1024, (r+1)*1024) of each workload (fixtures.shard; the
N>1 host logic is covered by tests/test_multiproc.py with gloo, world size 2).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fixtures as fx  # noqa: E402

METRIC = "coded query groups/sec (k=10, CIFAR-shape) at 1/2/4/8 B200; % tensor/HBM peak"
UNIT = "groups/s"
NBUF = 4


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


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


# ----------------------------------------------------------------------------- oracle leg
def oracle_sample(cfg, params, x, drop, groups):
    import oracle
    t0 = time.perf_counter()
    ref = oracle.serve_group(cfg.arch, params, x[groups], drop[groups], learned=bool(cfg.arch.encoder),
                             fp_iters=cfg.arch.fp_iters)
    dt = time.perf_counter() - t0
    return ref, dt


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
    step; encode exact (X2 reduce + h^-1 + h on the parity GPU) or learned (encoder on the parity
    GPU); decode as a masked NCCL reduce-scatter (paper_2106_06445_b200/workers.py)."""
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
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2106_06445_b200 import codedinv as ci
    from paper_2106_06445_b200.workers import GpuCompute, serve_workers
    arch = cfg.arch
    learned = args.encode == "learned"
    model = ci.Model(arch, fx.make_weights(arch, cfg.seed_w), args.precision, device=local)
    comp = GpuCompute(model, k, B)
    dev = torch.device("cuda", local)
    x = fx.make_inputs(arch, B, k, cfg.seed_x)
    drop = torch.from_numpy(fx.make_drops(B, k, cfg.seed_drop)).to(dev)
    x_slot = torch.from_numpy(np.ascontiguousarray(x[:, rank])).to(dev) if rank < k else None
    x_all = torch.from_numpy(x).to(dev) if rank == k else None
    step = lambda: serve_workers(comp, dist, rank, world, k, drop, x_slot=x_slot, x_all=x_all, learned=learned)
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
    t = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": B * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "none (fixed 8-worker partition)",
                          "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
                          "config": {"workload": "C5", "k": k, "groups_per_step": B, "encode": args.encode,
                                     "parallelism": "worker-per-GPU (k=7 main + 1 parity), NCCL reduce / "
                                                    "reduce-scatter decode"}}), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- our path
def relerr(a, ref):
    a = np.asarray(a, np.float64).reshape(-1, np.shape(ref)[-1])
    r = np.asarray(ref, np.float64).reshape(-1, np.shape(ref)[-1])
    return float(np.max(np.max(np.abs(a - r), 1) / np.maximum(np.max(np.abs(r), 1), 1e-30)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32", "simt"])
    ap.add_argument("--config", default="C3", choices=["C3", "C4", "C5", "C2", "C1", "C3R"])
    ap.add_argument("--encode", default="exact", choices=["exact", "learned"], help="C5 parity encode mode")
    ap.add_argument("--ref-groups", type=int, default=8, help="oracle sample groups per step")
    ap.add_argument("--cpu-groups", type=int, default=8, help="oracle sample for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other-precision throughput line item")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the standalone HBM / online-decode / label-generation line items")
    ap.add_argument("--inflight", type=int, default=2, choices=[1, 2, 3, 4],
                    help="request batches in flight (2: consecutive steps alternate between two CUDA streams)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    if args.config == "C5":
        return run_c5(args, rank, world, local)
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2106_06445_b200 import codedinv as ci

    cfg = fx.CONFIGS[args.config]
    arch, k, B = cfg.arch, cfg.k, cfg.B
    d, din = arch.d, arch.in_c * arch.in_h * arch.in_w
    learned = bool(arch.encoder)
    params = fx.make_weights(arch, cfg.seed_w)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    # group-sharded data parallelism: rank r serves global groups [r*B, (r+1)*B) of each of
    # NBUF rotating global workloads (counter-based slices: no rank generates others' groups)
    b0, b1 = fx.shard(rank, world, B)
    xs = [torch.from_numpy(fx.make_inputs_slice(arch, b0, b1, k, cfg.seed_x + 7919 * i)).to(dev)
          for i in range(NBUF)]
    drops = [torch.from_numpy(fx.make_drops_slice(b0, b1, k, cfg.seed_drop + 7919 * i)).to(dev)
             for i in range(NBUF)]
    hs = [torch.empty(B, k, d, device=dev) for _ in range(NBUF)]
    ps = [torch.empty(B, d, device=dev) for _ in range(NBUF)]
    ncls = sum(arch.heads)
    lg = [torch.empty(B * k * ncls, device=dev) for _ in range(NBUF)]
    lb = [torch.empty(B * k * len(arch.heads), dtype=torch.int32, device=dev) for _ in range(NBUF)]

    def run_mode(precision, steps, warmup, measure=True, nin=1, prof=None):
        """measure: sample clocks; prof: per-launch CUDA events on the stage kernel (needs nin=1)."""
        prof = (measure and nin == 1) if prof is None else prof
        model = ci.Model(arch, params, precision, device=local)
        wss = [model.workspace(k, B) for _ in range(nin)]
        ws = wss[0]
        streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nin - 1)]

        def serve(i):
            j = i % NBUF
            sidx = i % nin
            st = streams[sidx]
            model.ci_serve_group(xs[j], drops[j], hs[j], ps[j], wss[sidx], logits=lg[j], labels=lb[j],
                                 learned=learned, stream=st)

        for s_ in streams[1:]:
            s_.wait_stream(stream)
        for i in range(warmup):
            serve(i)
        torch.cuda.synchronize()
        ci.ci_test_prof_read()
        ci.ci_test_launch_count(reset=True)
        sampler = ClockSampler(local)
        if measure:
            sampler.start()
            time.sleep(0.2)
        ci.ci_test_prof_enable(prof and nin == 1)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s_ in streams[1:]:
            s_.wait_stream(stream)
        for i in range(steps):
            serve(i)
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
        kms, kl, kfl = ci.ci_test_prof_read()
        for w_ in wss:
            model.ci_check(w_)
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return dict(model=model, ws=ws, ms=ms, clocks=clocks, launches=launches,
                    kms=kms, klaunch=kl, kflops=kfl)

    peaks, peak_src = load_peaks()
    main_run = run_mode(args.precision, args.steps, args.warmup, nin=args.inflight)
    ms_step = main_run["ms"] / args.steps
    value = world * B * args.steps / (main_run["ms"] / 1e3)
    # per-launch kernel timing needs one stream: a separate single-stream pass when inflight > 1
    prof_run = main_run if args.inflight == 1 else run_mode(args.precision, max(3, args.steps // 2), 3,
                                                            measure=False, nin=1, prof=True)

    # --- roofline of the dominant kernel (fused tcgen05 stage kernel), live CUDA events
    kms, kfl, kl = prof_run["kms"], prof_run["kflops"], prof_run["klaunch"]
    stage_ms, stage_fl = sum(kms), sum(kfl)
    roofline = None
    kernels = {}
    if stage_ms > 0:
        achieved = stage_fl / (stage_ms / 1e3) / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        mult = 3 if args.precision == "fp32" else 1
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(f"k_stage_{args.precision}")
            except Exception:
                traffic = None
        roofline = {"bound": "tensor", "kernel": "k_stage (fused coupling stage, tcgen05)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "peak_source": f"{peak_src} bf16_tflops_sustained (dense bf16 cuBLAS, 4 s loop)",
                    "frac_of_burst": achieved / peaks["bf16_tflops"],
                    "issued_mma_multiplier": mult, "traffic": traffic,
                    "share_of_step": stage_ms / prof_run["ms"],
                    "measured_in": "single-stream pass" if args.inflight > 1 else "timed region"}
        for s in range(4):
            if kl[s]:
                kernels[f"k_stage[s{s}]"] = {"launches": kl[s], "ms_per_launch": kms[s] / kl[s],
                                             "tflops": kfl[s] / (kms[s] / 1e3) / 1e12,
                                             "frac_of_peak": kfl[s] / (kms[s] / 1e3) / 1e12 / peak}

    # --- HBM roofline of encode-mean / decode: standalone, L2-cold, 1.1 GB working set
    hbm = {}
    if rank == 0 and not args.no_extras:
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
        del Hb, Pb, flush
        # online decoding (f2): the wave that completes every group (the only
        # decode work on the critical path) vs the batch decode, 1024 groups, L2 flushed
        online = {}
        flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)

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
        del flush

    # --- e2e through the host-buffer C-ABI call (pinned host memory, copies in the region)
    e2e = None
    if not args.no_e2e:
        model = main_run["model"]
        nin = args.inflight
        # one host workspace + pinned output set per in-flight call (inputs are shared, read-only)
        xh = torch.from_numpy(fx.make_inputs_slice(arch, b0, b1, k, cfg.seed_x)).pin_memory()
        dh = torch.from_numpy(fx.make_drops_slice(b0, b1, k, cfg.seed_drop)).pin_memory()
        sets = []
        for _ in range(nin):
            hh = torch.empty(B, k, d).pin_memory()
            ph = torch.empty(B, d).pin_memory()
            lgh = torch.empty(B * k * ncls).pin_memory()
            lbh = torch.empty(B * k * len(arch.heads), dtype=torch.int32).pin_memory()
            sets.append(((xh.numpy(), dh.numpy(), hh.numpy(), ph.numpy(), lgh.numpy(), lbh.numpy()),
                         model.workspace(k, B, host=True)))
        estreams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nin - 1)]

        def e2e_call(i):
            a_h, w_h = sets[i % nin]
            model.ci_serve_group_host(*a_h, w_h, learned=learned, stream=estreams[i % nin], sync=(nin == 1))

        for i in range(2 * nin):
            e2e_call(i)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e_steps = max(3, min(args.steps, 10))
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
        ems = a_.elapsed_time(b_)
        for _, w_h in sets:
            model.ci_check(w_h)
        if dist:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        hh, ph, lgh, lbh = (torch.from_numpy(a) for a in sets[0][0][2:])
        e2e = {"value": world * B * e_steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(xh.numel() * 4 + dh.numel() * 4),
               "d2h_bytes_per_step": int(hh.numel() * 4 + ph.numel() * 4 + lgh.numel() * 4 + lbh.numel() * 4),
               "steps": e_steps, "inflight": nin,
               "note": "ci_serve_group_host(_async): pinned H2D of x+drop, D2H of h_out, h_parity, logits, "
                       "labels inside the device-timed region; calls alternate over `inflight` streams"}
        del sets

    # --- bulk encoder-label generation (f4; "draw k random inputs and compute
    #     labels f^-1(sum_j c_j f(x_j)) ... 50,000 times"): h on the k inputs + mean + h^-1 per
    #     tuple, exact encode, 1024 tuples per call
    label_gen = None
    if not learned and rank == 0 and not args.no_extras:
        model = main_run["model"]
        wsl = main_run["ws"]
        hl = torch.empty(B, k, d, device=dev)
        xl = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device=dev)
        def gen(j):
            model.ci_forward_h(xs[j].view(B * k, arch.in_c, arch.in_h, arch.in_w), hl.view(B * k, d), wsl)
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
                     "seconds_for_50000": 50000 / (B / (lms / 1e3)),
                     "note": "exact (x-tuple, h^-1(mean h)) training pairs for the learned encoder"}
        del hl, xl

    # --- encoding overhead vs k (Figs. 6-7 analogue): encoder time / time of
    #     h on the k main queries, batch of 1024 groups, learned encoder only
    enc_over = None
    if learned and rank == 0:
        model = main_run["model"]
        enc_over = {}
        for kk in (2, 4, 10):
            xk = torch.from_numpy(fx.make_inputs_slice(arch, 0, B, kk, cfg.seed_x)).to(dev)
            wsk = model.workspace(kk, B)
            hk = torch.empty(B * kk, d, device=dev)
            xpk = torch.empty(B, arch.in_c, arch.in_h, arch.in_w, device=dev)
            def timed(fn, reps=5):
                fn(); torch.cuda.synchronize()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for _ in range(reps):
                    fn()
                b_.record(stream)
                torch.cuda.synchronize()
                return a_.elapsed_time(b_) / reps
            t_enc = timed(lambda: model.ci_encode(None, xpk, wsk, x=xk, learned=True))
            t_h = timed(lambda: model.ci_forward_h(xk.reshape(B * kk, arch.in_c, arch.in_h, arch.in_w), hk, wsk))
            enc_over[str(kk)] = {"encoder_ms": t_enc, "h_ms": t_h, "overhead": t_enc / t_h}
            del xk, wsk, hk, xpk

    # --- other precision (throughput line item, same workload)
    alt = None
    if not args.no_alt:
        other = "fp32" if args.precision == "bf16" else "bf16"
        r2 = run_mode(other, max(3, args.steps // 3), 3, measure=False, nin=args.inflight)
        alt = {"precision": other, "value": world * B * max(3, args.steps // 3) / (r2["ms"] / 1e3),
               "ms_per_step": r2["ms"] / max(3, args.steps // 3)}
        del r2

    # --- numerics + cpu_baseline: oracle on a bounded sample of buffer 0's groups (rank 0)
    cpu = None
    numerics = None
    if rank == 0 and not args.no_cpu_baseline:
        xs0 = xs[0].cpu().numpy()
        dr0 = drops[0].cpu().numpy()
        model = main_run["model"]
        ws = main_run["ws"]
        model.ci_serve_group(xs[0], drops[0], hs[0], ps[0], ws, logits=lg[0], labels=lb[0], learned=learned)
        torch.cuda.synchronize()
        rng = np.random.default_rng(2106)
        S = args.cpu_groups
        groups = np.sort(rng.choice(B, S, replace=False))
        ref, dt = oracle_sample(cfg, params, xs0, dr0, groups)
        cores = os.cpu_count()
        cpu = {"value": S / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{S} seeded groups of {cfg.name} (k={k}: {S * (k + 2)} h-equivalents, f64 C "
                         f"oracle, pthreads over images), wall {dt:.1f} s"}
        R = hs[0].cpu().numpy()[groups]
        P = ps[0].cpu().numpy()[groups]
        L = lg[0].cpu().numpy()[:B * k * arch.heads[0]].reshape(B, k, arch.heads[0])[groups]
        lab = lb[0].cpu().numpy()[:B * k].reshape(B, k)[groups]
        bi = np.arange(S)
        numerics = {"groups_checked": S, "precision": args.precision,
                    "max_rel_err_features": relerr(R, ref["R"]),
                    "max_rel_err_decoded": relerr(R[bi, dr0[groups]], ref["R"][bi, dr0[groups]]),
                    "max_rel_err_parity": relerr(P, ref["P"]),
                    "max_rel_err_logits": relerr(L, ref["logits"][0]),
                    "label_agreement": float(np.mean(lab == ref["labels"][0])),
                    "label_agreement_decoded": float(np.mean(lab[bi, dr0[groups]] == ref["labels"][0][bi, dr0[groups]])),
                    "tolerance": 1e-3}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": {"bf16": "bf16", "fp32": "bf16x3", "simt": "f32"}[args.precision],
                "data": "synthetic",
                "config": {"workload": cfg.name, "k": k, "groups_per_gpu": B, "global_groups": B * world,
                           "queries_per_group": k + 1, "image": "3x32x32",
                           "arch": fx.arch_summary(arch),
                           "encode": "exact h^-1(mean h)", "precision": args.precision,
                           "parallelism": f"group-sharded x{world}",
                           "l2": f"inputs rotate over {NBUF} resident buffer sets (x+outputs ~1 GB > L2)",
                           "inflight": args.inflight},
                "roofline": roofline, "kernels": kernels, "hbm": hbm,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": main_run["launches"], "clocks": main_run["clocks"],
                "numerics": numerics, "alt_precision": alt}
        if enc_over is not None:
            line["encoder_overhead"] = enc_over
            line["config"]["encode"] = "learned encoder (Arch E), heads 10 + 2"
        if label_gen:
            line["label_generation"] = label_gen
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
