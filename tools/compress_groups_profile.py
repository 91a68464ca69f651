"""cProfile of a steady-state compress_groups call (diagnostic)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0], "--groups", sys.argv[1] if len(sys.argv) > 1 else "1024"]

import bench  # noqa: E402
from paper_2008_06972_b200 import codec, synth  # noqa: E402

args = bench.parse()
sensor, n, tile, tau, scene, G = bench.workload(args)
cfg = bench.codec_config(sensor, n, tile, tau)
groups, poses = [], []
for g in range(G):
    grp = synth.make_group(bench.group_seed(0, g, 4), n, sensor, **scene)
    groups.append(grp.clouds)
    poses.append(grp.poses)
codec.compress_groups(groups, cfg, poses)
pr = cProfile.Profile()
pr.enable()
codec.compress_groups(groups, cfg, poses)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
