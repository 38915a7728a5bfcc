"""Aggregate ncu source-page stall samples / instructions into line-range regions of one file."""
import csv
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = [tuple(map(int, r.split("-"))) + (n,) for r, n in (x.split(":") for x in sys.argv[3:])]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr = None, None
agg = {}
tot_s = tot_i = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        ln = int(r[0])
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ins = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    tot_s += smp
    tot_i += ins
    key = cur_file
    if cur_file == fname:
        for a, b, n in ranges:
            if a <= ln <= b:
                key = f"{fname}:{n}"
                break
    s = agg.setdefault(key, [0, 0])
    s[0] += smp
    s[1] += ins
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:40s} samples {100 * v[0] / tot_s:5.1f}%  inst {100 * v[1] / max(tot_i, 1):5.1f}%")
