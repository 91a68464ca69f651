"""Host-side cost of the device-resident decode call on the bench workload
(diagnostic): wall time per call and a cProfile of one call.

    python tools/decode_host_profile.py [groups]
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_06972_b200 import Encoder, _native  # noqa: E402
from paper_2008_06972_b200.decode import Decoder  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    sys.argv = [sys.argv[0], "--groups", str(G)]
    args = bench.parse()
    sensor, n, tile, tau, scene, G = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    L = _native.load(require_device=True)
    d_pts, off, xf = bench.make_inputs(args, 0, torch.device("cuda", 0))
    enc = Encoder(cfg)
    enc.encode_device(G, d_pts.data_ptr(), off, xf, None)
    torch.cuda.synchronize()
    off_b, _ = enc.blob_layout()
    dptr = L.stpc_result_device_blobs(enc.handle)
    offs = np.ascontiguousarray(off_b[:G + 1], np.int64)
    dec = Decoder()
    for _ in range(3):
        dec.decode(dptr, offs, True, keep_on_device=True)
    t = time.perf_counter()
    for _ in range(5):
        dec.decode(dptr, offs, True, keep_on_device=True)
    print(f"decode: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms per call")
    pr = cProfile.Profile()
    pr.enable()
    dec.decode(dptr, offs, True, keep_on_device=True)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
