"""Per-source-line warp-stall samples of an ncu report (source page, cuda+sass):
python scripts/ncu_lines.py REPORT.ncu-rep [N]"""
import csv, io, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = []
tot = 0
for r in rows:
    if len(r) != len(hdr) or r[0] in ("", "Line No"):
        continue
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    st = sorted(((int(r[hdr.index(c)] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    lines.append((s, r[0], r[1].strip()[:90], st))
lines.sort(reverse=True)
print("total samples", tot)
for s, ln, src, st in lines[:top]:
    print(f"{s:7d} {100.0*s/tot:5.1f}% L{ln:>5} {src:90s} {' '.join(f'{n}:{v}' for v, n in st if v)}")
if len(sys.argv) > 3:   # region sums: name:lo-hi,...
    for spec in sys.argv[3].split(","):
        name, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        s = sum(x[0] for x in lines if x[1].isdigit() and lo <= int(x[1]) <= hi)
        print(f"region {name:10s} L{lo}-{hi}: {s} ({100.0*s/tot:.1f}%)")
