"""Summarise ncu outputs for profiles/ (run here, on the files gpurun brings back).

    python tools/ncu_summary.py launches gpurun_out/launches.csv      # per-kernel time shares
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep          # key metrics per captured kernel
"""
import collections
import csv
import json
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"^_ZN4stpc\d+", "", d["Kernel Name"])
        name = re.sub(r"\(.*", "", name)
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[d["Metric Unit"]]
        v = float(d["Metric Value"].replace(",", "")) * scale
        tot[name] = tot.get(name, 0.0) + v
        cnt[name] += 1
    T = sum(tot.values())
    out = [{"kernel": k, "launches": cnt[k], "ms": round(v, 4), "share": round(v / T, 4)}
           for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]
    return {"total_ms": round(T, 3), "kernels": out}


WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__registers_per_thread": "registers",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "")), "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for m, nm in WANT.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    k[nm] = float(d[m].replace(",", ""))
                    k[nm + "_unit"] = u.get(m, "")
                except ValueError:
                    pass
        res.append(k)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
