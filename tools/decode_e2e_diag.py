"""Host-side phase timing of decompress_many on bench blobs (diagnostic).

    python tools/decode_e2e_diag.py [groups]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_06972_b200 import Encoder, _native  # noqa: E402
from paper_2008_06972_b200 import decode as D  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    sys.argv = [sys.argv[0], "--groups", str(G)]
    args = bench.parse()
    sensor, n, tile, tau, scene, G = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    d_pts, off, xf = bench.make_inputs(args, 0, torch.device("cuda", 0))
    enc = Encoder(cfg)
    enc.encode_device(G, d_pts.data_ptr(), off, xf, None)
    torch.cuda.synchronize()
    blobs = enc.blobs()
    del d_pts
    D.decompress_many(blobs)
    dec = D.get_decoder()
    for _ in range(3):
        t1 = time.perf_counter()
        clouds, reps, errs = dec.decode(0, None, False, host_blobs=blobs)
        t2 = time.perf_counter()
        tm = reps[0].timings
        npts = sum(c.shape[0] for cl in clouds for c in cl)
        print(f"decompress_many {1e3*(t2-t1):.1f} ms (deserialize {1e3*tm['deserialize']:.1f}, "
              f"points {1e3*tm['reconstruct']:.1f})  points {npts}  bytes out {24*npts/1e9:.2f} GB  "
              f"-> {len(blobs) * 8 / (t2 - t1):.0f} frames/s")
    # pinned vs pageable D2H of the same bytes
    nbytes = 24 * npts
    dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    for pin in (False, True):
        h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=pin)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.copy_(dev)
        torch.cuda.synchronize()
        print(f"D2H {nbytes/1e9:.2f} GB pinned={pin}: {1e3*(time.perf_counter()-t0):.1f} ms")
    t0 = time.perf_counter()
    x = np.empty(nbytes // 8)
    x[::512] = 0.0
    print(f"np.empty + first touch {nbytes/1e9:.2f} GB: {1e3*(time.perf_counter()-t0):.1f} ms")


if __name__ == "__main__":
    main()
