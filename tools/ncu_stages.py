"""Per-stage ncu metrics of one encode step, stamped with the source hash.

On the GPU box (after the same bench command has exited 0 without ncu):

    ncu --clock-control none --kernel-name-base demangled -k regex:stpc:: \\
        --metrics <METRICS below, comma-joined> --csv --log-file gpurun_out/stages.csv \\
        python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-decode --no-parity

Here:

    python tools/ncu_stages.py gpurun_out/stages.csv profiles/r2_ncu_stages.json

The launches of the one encode call map onto the pipeline stages in launch
order (encoder.cu encode_impl); bench.py reads the JSON for `traffic` and the
issue-rate fields only while its `source_hash` equals the current sources'.
"""

from __future__ import annotations

import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def kernel_stage(name: str, seen: dict) -> str:
    """Stage of a launch (encoder.cu encode_impl order); `seen` counts launches."""
    n = seen.get(name, 0)
    seen[name] = n + 1
    if "fill_u64" in name:  # the first call's +inf grid fill (steady-state calls get it from the previous pack)
        return "other"
    if "convert" in name:
        return "convert"
    if "emit" in name:  # before "bitmap": emit_bitmaps_kernel is part of emit
        return "emit"
    if "bitmap" in name:
        return "bitmaps"
    if "start_tiles" in name:
        return "start_key" if n == 0 else "start_p"
    if "fit_pair" in name or "fit_rows" in name:
        return "fit_key" if n == 0 else "fit_p"
    if "refit" in name or "chain_bytes" in name:
        return "refit"
    if "rowstats" in name or "plan" in name or "group_scan" in name:
        return "plan"
    if "emit" in name:
        return "emit"
    if "histogram" in name or "code_lengths" in name:
        return "huffman"
    if "pack" in name:
        return "pack"
    if "crc" in name:
        return "crc"
    return "other"


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        L = launches.setdefault(key, {"kernel": d["Kernel Name"]})
        v = d["Metric Value"].replace(",", "")
        try:
            val = float(v) * SCALE.get(d.get("Metric Unit", ""), 1.0)
        except ValueError:
            continue
        L[d["Metric Name"]] = val
    return [launches[k] for k in sorted(launches)]


def main():
    src, out = sys.argv[1], sys.argv[2]
    from paper_2008_06972_b200 import build

    launches = parse(src)
    seen, stages = {}, {}
    for L in launches:
        base = re.sub(r"^_ZN4stpc\d+", "", L["kernel"])
        base = re.sub(r"^void\s+", "", base)
        base = re.sub(r"^stpc::", "", base)
        base = re.match(r"[A-Za-z_0-9]+", base).group(0)
        st = kernel_stage(base, seen)
        S = stages.setdefault(st, {"kernels": {}, "dram_bytes": 0.0, "warp_instructions": 0.0, "ms": 0.0})
        S["kernels"][base] = S["kernels"].get(base, 0) + 1
        S["dram_bytes"] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        S["warp_instructions"] += L.get("smsp__inst_executed.sum", 0)
        ms = L.get("gpu__time_duration.sum", 0)
        S["ms"] += ms
        # time-weighted per-launch rates
        for k, nm in (("sm__inst_executed.avg.per_cycle_active", "ipc"),
                      ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
                      ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
                      ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
                      ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct")):
            if k in L:
                S.setdefault("_w_" + nm, 0.0)
                S["_w_" + nm] += L[k] * ms
    for S in stages.values():
        for k in [k for k in S if k.startswith("_w_")]:
            S[k[3:]] = round(S.pop(k) / S["ms"], 3) if S["ms"] else None
        S["issue_frac"] = round(S["ipc"] / 4.0, 4) if S.get("ipc") is not None else None
        S["ms"] = round(S["ms"], 4)
    res = {"source_hash": build.source_hash(), "capture": os.path.basename(src),
           "command": "ncu --metrics " + ",".join(METRICS) + " python bench.py --steps 1 --warmup 0 --no-e2e "
                      "--no-cpu --no-decode --no-parity (one encode step of the bench workload)",
           "note": "ncu times are cold-cache and serialised: compare shares, not absolutes",
           "stages": stages}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: {kk: v[kk] for kk in ("ms", "dram_bytes", "ipc", "issue_frac")} for k, v in stages.items()},
                     indent=0))


if __name__ == "__main__":
    main()
