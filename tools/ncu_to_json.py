"""Turn one `ncu --set full` capture of the hot sweep kernel into
profiles/sim_kernel_ncu.json, the file bench.py's `roofline` reads for its
measured-DRAM and issue-slot fractions (`traffic`, `dram_frac`, `issue_frac`).

usage: python tools/ncu_to_json.py REPORT.ncu-rep N_REQUESTS CELLS [OUT.json]"""
import csv
import json
import os
import subprocess
import sys


def raw(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [dict(zip(h, v)) for v in rows[2:]], dict(zip(h, u))


def num(s: str) -> float:
    return float(s.replace(",", ""))


def main() -> None:
    rep, n_req, cells = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    dst = sys.argv[4] if len(sys.argv) > 4 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
        "sim_kernel_ncu.json")
    launches, units = raw(rep)
    # the hot kernel: the longest sl_sim_fast_kernel launch in the capture
    cand = [d for d in launches if "sl_sim_fast_kernel" in d.get("Kernel Name", "")]
    d = max(cand, key=lambda x: num(x["gpu__time_duration.sum"]))
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9, "s": 1e9}
    t_ns = num(d["gpu__time_duration.sum"]) * scale[units["gpu__time_duration.sum"]]
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    dram = sum(num(d[k]) * bscale[units[k]] for k in ("dram__bytes_read.sum",
                                                      "dram__bytes_write.sum"))
    hz = num(d["sm__cycles_elapsed.avg.per_second"]) * {
        "cycle/second": 1.0, "cycle/msecond": 1e3, "cycle/usecond": 1e6,
        "cycle/nsecond": 1e9, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}[units["sm__cycles_elapsed.avg.per_second"]]
    out = {
        "kernel": d["Kernel Name"],
        "n_requests": n_req,
        "cells": cells,
        "gpu_time_ns": t_ns,
        "dram_bytes": dram,
        "inst_executed": num(d["smsp__inst_executed.sum"]),
        "sm_clock_hz": hz,
        "sms": int(num(d["device__attribute_multiprocessor_count"])),
        "issue_active_pct": num(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "warps_active_pct": num(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "registers": int(num(d["launch__registers_per_thread"])),
        "source": os.path.basename(rep) + " (ncu --set full --clock-control none, one launch)",
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
