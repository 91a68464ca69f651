"""Phase breakdown of the GPU decoder on the bench workload (diagnostic).

    python tools/decode_diag.py [groups]
"""

import ctypes
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
    dev = torch.device("cuda", 0)
    d_pts, off, xf = bench.make_inputs(args, 0, dev)
    enc = Encoder(cfg)
    enc.encode_device(G, d_pts.data_ptr(), off, xf, None)
    torch.cuda.synchronize()
    off_b, len_b = enc.blob_layout()
    dptr = L.stpc_result_device_blobs(enc.handle)
    offs = np.ascontiguousarray(off_b[:G + 1], np.int64)
    dec = D.Decoder()
    for rep in range(3):
        t = [time.perf_counter()]
        status = np.zeros(G, np.int32)
        _native.check(L.stpc_decoder_load(dec.h, dptr, 1, offs.ctypes.data, G, status.ctypes.data, None))
        t.append(time.perf_counter())
        raw_len = np.zeros(G, np.int64)
        cap = 57 + 48 * 16
        heads = np.zeros((G, cap), np.uint8)
        _native.check(L.stpc_decoder_heads(dec.h, cap, heads.ctypes.data, raw_len.ctypes.data, None))
        t.append(time.perf_counter())
        cfgs = [D._config(heads[i].tobytes(), int(raw_len[i])) for i in range(G)]
        t.append(time.perf_counter())
        good, bad = D._transforms_batch(heads, raw_len, list(range(G)), n)
        xfi = [good[i] for i in range(G)]
        t.append(time.perf_counter())
        c = cfgs[0]
        geom = _native.StpcDecodeGeom(c["w"], c["h"], c["tile_w"], c["tile_h"], n, c["k_index"],
                                      c["range_quant"], 200.0)
        st, ct, sp, cp = (np.ascontiguousarray(a) for a in
                          D.ray_trig_tables(c["w"], c["h"], c["theta_r"], c["phi_r"], c["phi_offset"]))
        sel = np.arange(G, dtype=np.int32)
        X = np.ascontiguousarray(np.concatenate(xfi))
        counts = np.zeros(G * n, np.int64)
        pst = np.zeros(G, np.int64)
        failed = np.zeros(G, np.int64)
        t.append(time.perf_counter())
        _native.check(L.stpc_decoder_frames(dec.h, ctypes.byref(geom), sel.ctypes.data, G, st.ctypes.data,
                                            ct.ctypes.data, sp.ctypes.data, cp.ctypes.data, X.ctypes.data,
                                            counts.ctypes.data, pst.ctypes.data, failed.ctypes.data, None))
        t.append(time.perf_counter())
        _native.check(L.stpc_decoder_points(dec.h, None, 1, 0, None))
        t.append(time.perf_counter())
        names = ["load(crc+huff)", "heads", "config", "transforms", "prep", "frames", "points"]
        print(" ".join(f"{nm}={1e3 * (b - a):.2f}ms" for nm, a, b in zip(names, t[:-1], t[1:])),
              f"total={1e3 * (t[-1] - t[0]):.1f}ms pts={int(counts.sum())} err={int((pst != 0).sum())}")


if __name__ == "__main__":
    main()
