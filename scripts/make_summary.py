"""Regenerate profiles/r01_summary.md (+ bench JSON copies, traffic.json) from the gpurun_out/
artifacts of scripts/gpu_refresh.sh."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
for src, dst in (("bench_bf16", "bench_bf16"), ("bench_fp32", "bench_fp32"), ("bench_c4", "bench_c4"),
                 ("bench_c3r", "bench_c3r"), ("bench_ref", "bench_reference")):
    shutil.copy(os.path.join(G, src + ".json"), os.path.join(P, f"{tag}_{dst}.json"))
npass = open(os.path.join(G, "pytest_gpu.log")).read().strip().splitlines()[-1]

rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    agg[r[ki][:78]][0] += 1
    agg[r[ki][:78]][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
launch = ["| kernel | launches | total (ns) | share |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    launch.append(f"| `{k}` | {v[0]} | {v[1]:,.0f} | {v[1] / tot * 100:.1f}% |")

raw = subprocess.run(["ncu", "-i", os.path.join(G, f"prof_stage_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
R = list(csv.reader(raw.splitlines()))
H = R[0]
c = H.index
full = ["| kernel | duration (ms) | DRAM read MB | DRAM write MB | tensor pipe active % | SMEM->tensor active % | SM throughput % |",
        "|---|---|---|---|---|---|---|"]
traffic = []
for r in R[2:]:
    rd, wr = float(r[c("dram__bytes_read.sum")]), float(r[c("dram__bytes_write.sum")])
    traffic.append(rd + wr)
    full.append(f"| `{r[c('Kernel Name')][:52]}` | {float(r[c('gpu__time_duration.sum')]):.3f} | {rd:.1f} | {wr:.1f} | "
                f"{float(r[c('TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed')]):.1f} | "
                f"{float(r[c('sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')]):.1f} | "
                f"{float(r[c('sm__throughput.avg.pct_of_peak_sustained_elapsed')]):.1f} |")
json.dump({"k_stage_bf16_launches_MB": traffic, "k_stage_bf16": sum(traffic) / len(traffic) * 1e6,
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per k_stage launch (bytes), mean of the 3 "
                   "main-forward stage launches (10240 images), ncu --set full (scripts/gpu_refresh.sh)"},
          open(os.path.join(P, "traffic.json"), "w"), indent=1)

J = lambda n: json.load(open(os.path.join(P, f"{tag}_{n}.json")))
b, f, c4, cr, ref = J("bench_bf16"), J("bench_fp32"), J("bench_c4"), J("bench_c3r"), J("bench_reference")
k = b["kernels"]
od = b["hbm"]["online_decode"]["per_k"]
txt = f"""# Round 1 profile summary (B200, `scripts/gpu_refresh.sh` + `scripts/make_summary.py`, one box)

All numbers come from one `gpurun` call: `pytest -m gpu` ({npass}), the bench lines committed
next to this file (`{tag}_bench_*.json`), the ncu launch list and one `ncu --set full` capture of
the fused stage kernel.

## Live bench (CUDA events; default = 2 request batches in flight)
| workload | precision | groups/s | ms/step | e2e (host buffers) groups/s | stage-kernel TFLOP/s (frac of {b['roofline']['peak']} sustained) |
|---|---|---|---|---|---|
| C3 (Arch C, k=10, 1024 groups) | bf16 | {b['value']:,.0f} | {b['ms_per_step']:.2f} | {b['e2e']['value']:,.0f} | {b['roofline']['achieved']:.0f} ({b['roofline']['frac']:.3f}) |
| C3 | fp32 parity (bf16x3) | {f['value']:,.0f} | {f['ms_per_step']:.2f} | {f['e2e']['value']:,.0f} | {f['roofline']['achieved']:.0f}, 3 MMAs issued per product ({f['roofline']['frac']:.3f}) |
| C4 (learned encoder, heads 10+2) | bf16 | {c4['value']:,.0f} | {c4['ms_per_step']:.2f} | {c4['e2e']['value']:,.0f} | {c4['roofline']['achieved']:.0f} ({c4['roofline']['frac']:.3f}) |
| C3R (f1: i-ResNet residual, N=10 fixed-point h^-1) | bf16 | {cr['value']:,.0f} | {cr['ms_per_step']:.2f} | {cr['e2e']['value']:,.0f} | {cr['roofline']['achieved']:.0f} ({cr['roofline']['frac']:.3f}) |
| reference arm = f64 CPU oracle, {ref['cpu_baseline']['cores']} cores | f64 | {ref['value']:.2f} | {ref['ms_per_step']:.0f} | — | — |

Per-stage fused kernel (C3 bf16, single-stream profiled pass, avg over the 3 launch sizes):
s0 {k['k_stage[s0]']['tflops']:.0f} TFLOP/s ({k['k_stage[s0]']['frac_of_peak'] * 100:.1f}%), s1 {k['k_stage[s1]']['tflops']:.0f} ({k['k_stage[s1]']['frac_of_peak'] * 100:.1f}%),
s2 {k['k_stage[s2]']['tflops']:.0f} ({k['k_stage[s2]']['frac_of_peak'] * 100:.1f}%).  Clocks {b['clocks']['sm_mhz']:.0f}/{b['clocks']['sm_max_mhz']:.0f} MHz, throttle reasons {b['clocks']['reasons']}.
C3 bf16 numerics vs the oracle ({b['numerics']['groups_checked']} groups): decoded {b['numerics']['max_rel_err_decoded']:.2g}, parity {b['numerics']['max_rel_err_parity']:.2g},
logits {b['numerics']['max_rel_err_logits']:.2g}, labels {b['numerics']['label_agreement'] * 100:.2f}% (decoded slot {b['numerics']['label_agreement_decoded'] * 100:.1f}%).

HBM-bound kernels (standalone, 8192 groups, L2 flushed): decode {b['hbm']['decode']['achieved']:.0f} GB/s
({b['hbm']['decode']['frac'] * 100:.0f}% of measured {b['hbm']['decode']['peak']:.0f}), mean {b['hbm']['mean']['achieved']:.0f} GB/s ({b['hbm']['mean']['frac'] * 100:.0f}%).

Online decoding (f2, 1024 groups, L2 flushed), completing event vs batch decode:
""" + "\n".join(f"- {kk}: {v['completing_event_us']:.1f} us vs {v['batch_decode_us']:.1f} us" for kk, v in od.items()) + f"""

Bulk label generation (f4, exact (x-tuple, h^-1(mean h)) pairs): {b['label_generation']['pairs_per_s']:,.0f} pairs/s
(50,000 pairs in {b['label_generation']['seconds_for_50000']:.2f} s).

## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, `bench.py --steps 2 --warmup 1 --inflight 1`)
Cold-cache, serialised per-launch times; compare SHARES (the live bench puts the stage kernel at
{b['roofline']['share_of_step'] * 100:.1f}% of a step).  The capture also holds the bench's standalone L2-cold
decode/mean/online measurements and torch fills.

""" + "\n".join(launch) + """

## Full capture of the fused stage kernel (`ncu --set full -k regex:k_stage -s 9 -c 3`)
Main forward of 10240 images, one launch per stage (under ncu: cold, clocks not locked):

""" + "\n".join(full) + """

Algorithmic FLOPs per launch: n * 9 blocks * 36 * H*W * c * m (s0 0.326, s1 0.652, s2 1.305 TFLOP
for n = 10240).  DRAM traffic per launch (~200 MB) is the fp32 stage state in and out (126 MB)
plus weights from L2: the kernel is bound by tensor issue and epilogue/MMA serialisation, not DRAM.
Per-role cycle counters (`scripts/cycles.sh`) and ncu stall sampling locate the remaining gap:
the conv2 epilogue of block t must finish (tile by tile) before block t+1's conv1 can run, SS-mode
MMAs at N = 32 run at 40% of the tensor rate (s0, s1), and the padded raster wastes 14-36% of M.
"""
open(os.path.join(P, f"{tag}_summary.md"), "w").write(txt)
print(txt[:1500])
