"""Per-call latency of the drop-in compress() on one BASELINE configs[3] group
(diagnostic): wall time per call and a cProfile of one call.

    python tools/compress_latency.py [calls]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2008_06972_b200 import compress, synth  # noqa: E402


def main():
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    sys.argv = [sys.argv[0], "--groups", "1"]
    args = bench.parse()
    sensor, n, tile, tau, scene, _ = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    g = synth.make_group(bench.group_seed(0, 0, 4), n, sensor, device="cuda", **scene)
    compress(g.clouds, cfg, poses=g.poses)
    t = time.perf_counter()
    for _ in range(calls):
        compress(g.clouds, cfg, poses=g.poses)
    dt = (time.perf_counter() - t) / calls
    print(f"compress(): {dt * 1e3:.2f} ms per {n}-frame group ({n / dt:.0f} frames/s)")
    pr = cProfile.Profile()
    pr.enable()
    compress(g.clouds, cfg, poses=g.poses)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(14)


if __name__ == "__main__":
    main()
