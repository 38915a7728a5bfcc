"""Summarise an ncu report: key raw metrics + top source lines by stall samples."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    units = dict(zip(h, u))
    res = {k: (f"{d.get(k)} {units.get(k, '')}".strip() if d.get(k) is not None else None)
           for k in KEYS}
    stalls = {k.split("issue_stalled_")[1].replace("_per_issue_active.ratio", ""): float(x)
              for k, x in d.items() if "average_warps_issue_stalled" in k and x not in ("", "n/a")}
    return res, stalls


def lines(rep, n=30, steps=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, cur, agg, hdr = None, None, {}, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0] != "":
            try:
                cur = (cur_file, int(r[0]), r[1].strip()[:80])
            except ValueError:
                continue
            agg.setdefault(cur, [0, 0])
            continue
        if cur is None:
            continue
        try:
            agg[cur][0] += int(r[4])
            agg[cur][1] += int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            pass
    tot = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tot} warp-instructions {ti}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        per = f"{v[1] / steps:7.1f}/step" if steps else f"{100 * v[1] / ti:5.1f}%inst"
        print(f"{100 * v[0] / tot:5.1f}% {per} {k[0]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    rep = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else None
    r, st = raw(rep)
    for k, v in r.items():
        print(k, v)
    print("stalls/issue:", {k: round(v, 2) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v > 0.02})
    lines(rep, 40, steps)
