"""Timeline of the pipelined host encode (diagnostic): STPC_PIPE_TRACE=1
prints, per chunk, the H2D enqueue cost and the device times at which each
chunk's H2D and encode ended; this wrapper runs one warm call, then a traced
one, plus the pure H2D time of the same bytes.

    python tools/pipe_trace.py [groups] [chunks]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_06972_b200 import Encoder  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    if len(sys.argv) > 2:
        os.environ["STPC_PIPE_CHUNKS"] = sys.argv[2]
    sys.argv = [sys.argv[0], "--groups", str(G)]
    args = bench.parse()
    sensor, n, tile, tau, scene, G = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    d_pts, off, xf = bench.make_inputs(args, 0, torch.device("cuda"))
    enc = Encoder(cfg)
    s = torch.cuda.current_stream().cuda_stream
    h = torch.empty(d_pts.shape, dtype=torch.float32, pin_memory=True)
    h.copy_(d_pts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d_pts.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    print(f"pure H2D of {h.numel() * 4 / 1e9:.2f} GB: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
    hp = h.numpy()
    del d_pts
    torch.cuda.empty_cache()
    out = torch.empty(int(hp.nbytes // 8), dtype=torch.uint8, pin_memory=True).numpy()
    enc.encode_host(G, hp, off, xf, out, s)
    torch.cuda.synchronize()
    os.environ["STPC_PIPE_TRACE"] = "1"
    t0 = time.perf_counter()
    enc.encode_host(G, hp, off, xf, out, s)
    torch.cuda.synchronize()
    print(f"traced call: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)


if __name__ == "__main__":
    main()
