"""Device time of the decoder's load phase (CRC + Huffman) on the bench
workload, nothing after it (diagnostic; works with experimental builds that
leave the raw payloads unusable).

    python tools/huff_time.py [groups]
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
    dec = D.Decoder()
    status = np.zeros(G, np.int32)
    for rep in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _native.check(L.stpc_decoder_load(dec.h, dptr, 1, offs.ctypes.data, G, status.ctypes.data, None))
        torch.cuda.synchronize()
        print(f"load(crc+huff) {1e3 * (time.perf_counter() - t):.2f} ms, status nonzero {int((status != 0).sum())}")


if __name__ == "__main__":
    main()
