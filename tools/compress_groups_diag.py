"""Wall time of the public batch API compress_groups on bench groups (diagnostic).

    python tools/compress_groups_diag.py [groups]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2008_06972_b200 import compress_groups, synth  # noqa: E402
import bench  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    sys.argv = [sys.argv[0], "--groups", str(G)]
    args = bench.parse()
    sensor, n, tile, tau, scene, G = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    import torch

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = time.perf_counter()
    groups, poses = [], []
    for g in range(G):
        grp = synth.make_group(bench.group_seed(0, g, 4), n, sensor, device=dev, **scene)
        groups.append(grp.clouds)
        poses.append(grp.poses)
    print(f"generated {G} groups in {time.perf_counter() - t:.1f} s")
    compress_groups(groups[:2], cfg, poses[:2])
    for _ in range(3):
        t = time.perf_counter()
        blobs, reps = compress_groups(groups, cfg, poses)
        dt = time.perf_counter() - t
        print(f"compress_groups {G} groups: {dt * 1e3:.1f} ms -> {G * n / dt:.0f} frames/s; timings {reps[0].timings}")


if __name__ == "__main__":
    main()
