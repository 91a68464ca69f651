"""Steady-state per-call latency of the drop-in API, next to the oracle port.

For BASELINE configs[0], [1], [2] (one sweep point) and [4]: one seeded group,
3 warm-up calls (encoder pooled), then `calls` timed calls of
``compress(clouds, cfg, poses=...)`` -- host numpy clouds in, ``bytes`` out,
exactly the reference's call (pkg/tests/test_acceptance.py:171-194 times the
same call) -- and the single-core oracle port's per-call time on the same
input; likewise ``decompress(blob)`` (bytes in, float64 numpy clouds out)
beside the oracle decoder.  Also ``compress_groups`` on the configs[3] 1024-group batch (pageable
numpy in, ``bytes`` out).

    python tools/latency_table.py [--calls 20] [--out profiles/r2_latency.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import decode as odec  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2008_06972_b200 import compress, compress_groups, decompress, synth  # noqa: E402


def timed(fn, calls):
    out = []
    for _ in range(calls):
        t = time.perf_counter()
        fn()
        out.append((time.perf_counter() - t) * 1e3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--groups", type=int, default=1024)
    a = ap.parse_args()
    oracle.build()
    rows = []
    for cfg_id, label in ((1, "configs[0]"), (2, "configs[1]"), (3, "configs[2] (4x4, tau 0.1)"), (5, "configs[4]")):
        sensor, n, tile, tau, scene = synth.config_params(cfg_id)
        cfg = bench.codec_config(sensor, n, tile, tau)
        g = synth.make_group(bench.group_seed(0, 0, cfg_id), n, sensor, device="cuda", **scene)
        poses = g.poses if n > 1 else None
        call = lambda: compress(g.clouds, cfg, poses=poses)  # noqa: E731
        for _ in range(3):
            call()
        ms = timed(call, a.calls)
        ref_blob = oracle.compress(g.clouds, cfg, poses)[0]
        oms = timed(lambda: oracle.compress(g.clouds, cfg, poses), 3)
        row = {"config": label, "frames": n, "points": int(sum(c.shape[0] for c in g.clouds)),
               "compress_ms_median": round(statistics.median(ms), 3), "compress_ms_min": round(min(ms), 3),
               "compress_ms_p90": round(sorted(ms)[int(0.9 * (len(ms) - 1))], 3),
               "oracle_port_ms_1core": round(statistics.median(oms), 1),
               "speedup_vs_port": round(statistics.median(oms) / statistics.median(ms), 1),
               "identical": call()[0] == ref_blob, "calls": a.calls}
        for _ in range(3):
            decompress(ref_blob)
        dms = timed(lambda: decompress(ref_blob), a.calls)
        odms = timed(lambda: odec.decompress(ref_blob), 3)
        row.update({"decompress_ms_median": round(statistics.median(dms), 3),
                    "oracle_decoder_ms_1core": round(statistics.median(odms), 1),
                    "decompress_speedup_vs_port": round(statistics.median(odms) / statistics.median(dms), 1)})
        rows.append(row)
        print(json.dumps(row), flush=True)
    # the batch form through the public API
    sensor, n, tile, tau, scene = synth.config_params(4)
    cfg = bench.codec_config(sensor, n, tile, tau)
    groups, poses = [], []
    for gi in range(a.groups):
        grp = synth.make_group(bench.group_seed(0, gi, 4), n, sensor, device="cuda", **scene)
        groups.append(grp.clouds)
        poses.append(grp.poses)
    compress_groups(groups[:4], cfg, poses[:4])
    compress_groups(groups, cfg, poses)
    ms = timed(lambda: compress_groups(groups, cfg, poses), 3)
    row = {"config": f"configs[3] compress_groups, {a.groups} groups", "frames": a.groups * n,
           "points": int(sum(c.shape[0] for grp in groups for c in grp)),
           "compress_groups_ms_median": round(statistics.median(ms), 1),
           "frames_per_s": round(a.groups * n / (statistics.median(ms) / 1e3), 0),
           "input_bytes": int(sum(c.nbytes for grp in groups for c in grp))}
    rows.append(row)
    print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
