import os, sys, time
sys.path.insert(0, os.getcwd())
sys.argv = [sys.argv[0], "--groups", "1024"]
import numpy as np
import bench
from paper_2008_06972_b200 import synth, codec
args = bench.parse()
sensor, n, tile, tau, scene, G = bench.workload(args)
cfg = bench.codec_config(sensor, n, tile, tau)
groups, poses = [], []
for g in range(G):
    grp = synth.make_group(bench.group_seed(0, g, 4), n, sensor, **scene)
    groups.append(grp.clouds); poses.append(grp.poses)
print("contiguous:", all(c.flags['C_CONTIGUOUS'] for c in groups[0]), groups[0][0].dtype)
codec.compress_groups(groups[:2], cfg, poses[:2])
t = time.perf_counter(); fr, f64, counts = codec._frame_arrays([c for g in groups for c in g]); print("frame_arrays", time.perf_counter() - t)
t = time.perf_counter(); codec.compress_groups(groups, cfg, poses); print("compress_groups (1st)", time.perf_counter() - t)
os.environ["STPC_PIPE_TRACE"] = "1"
t = time.perf_counter(); codec.compress_groups(groups, cfg, poses); print("compress_groups (2nd)", time.perf_counter() - t)
