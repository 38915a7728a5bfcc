"""Per-source-line stall samples and instructions from an ncu report (cuda,sass source page).

usage: ncu_lines.py REP [N_TOP] [FILE:LO-HI=NAME ...]   (regions group lines of one file)"""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
regions = []
for a in sys.argv[3:]:
    f, rest = a.split(":")
    rng, name = rest.split("=")
    lo, hi = map(int, rng.split("-"))
    regions.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, f, agg = None, None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] != "":
        try:
            cur = (f, int(r[0]), r[1].strip()[:72])
        except ValueError:
            cur = None
        continue
    if cur is None:
        continue
    try:
        a = agg.setdefault(cur, [0, 0])
        a[0] += int(r[4])
        a[1] += int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts} warp-instructions {ti}")
grp = {}
for k, v in agg.items():
    name = k[0]
    for f, lo, hi, n in regions:
        if k[0] == f and lo <= k[1] <= hi:
            name = n
            break
    g = grp.setdefault(name, [0, 0])
    g[0] += v[0]
    g[1] += v[1]
for k, v in sorted(grp.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} samples {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
    print(f"{100 * v[0] / ts:5.1f}% {100 * v[1] / ti:5.1f}%i {k[0]}:{k[1]} {k[2]}")
