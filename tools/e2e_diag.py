"""Diagnose the e2e pipeline: device encode vs pure H2D vs pipelined host encode."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2008_06972_b200 import Encoder

class A: pass
a = A(); a.config = 4; a.groups = int(sys.argv[1]) if len(sys.argv) > 1 else 1024; a.tile = None; a.tau = None
sensor, n, tile, tau, scene, G = bench.workload(a)
cfg = bench.codec_config(sensor, n, tile, tau)
d_pts, off, xf = bench.make_inputs(a, 0, torch.device("cuda"))
enc = Encoder(cfg)
s = torch.cuda.current_stream()
enc.encode_device(G, d_pts.data_ptr(), off, xf, s.cuda_stream); torch.cuda.synchronize()
def t(fn, k=2):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
print("device encode ms", t(lambda: enc.encode_device(G, d_pts.data_ptr(), off, xf, s.cuda_stream)))
h = torch.empty(d_pts.shape, dtype=torch.float32, pin_memory=True); h.copy_(d_pts)
print("pure h2d ms", t(lambda: d_pts.copy_(h, non_blocking=True)))
hp = h.numpy()
o, ln = enc.blob_layout()
out = torch.empty(int(o[-1] * 1.3) + 4096, dtype=torch.uint8, pin_memory=True).numpy()
print("host encode pipelined ms", t(lambda: enc.encode_host(G, hp, off, xf, out, s.cuda_stream)))
print("host encode one-shot (no out) ms", t(lambda: enc.encode_host(G, hp, off, xf, None, s.cuda_stream), 1))
