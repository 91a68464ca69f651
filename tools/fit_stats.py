"""Chain-step statistics of the fit kernels on the bench workload (diagnostic).

    python tools/fit_stats.py [groups]

From the encoder's run buffers: runs per chain, run lengths, tile classes
(0 residual / 1 temporal / 2 fallback) for key and P frames, and the implied
number of chain steps.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_06972_b200 import Encoder, _native  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    sys.argv = [sys.argv[0], "--groups", str(G)]
    args = bench.parse()
    sensor, n, tile, tau, scene, G = bench.workload(args)
    cfg = bench.codec_config(sensor, n, tile, tau)
    d_pts, off, xf = bench.make_inputs(args, 0, torch.device("cuda", 0))
    enc = Encoder(cfg)
    L = _native.load()
    import ctypes
    dbg = getattr(L, "stpc_debug_fit_stats", None)
    if dbg is not None:
        L.stpc_debug_fit_stats_reset()
    enc.encode_device(G, d_pts.data_ptr(), off, xf, None)
    torch.cuda.synchronize()
    if dbg is not None:
        st = (ctypes.c_ulonglong * 8)()
        dbg(st)
        names = ["steps", "starts", "empty", "cert_checks", "weak_certs", "growth_tests", "growth_pass", "retest_fail"]
        print("fit counters (key + P):", {k: int(v) for k, v in zip(names, st)})
    F = G * n
    tx = -(-cfg.w // cfg.tile_w)
    ty = -(-cfg.h // cfg.tile_h)
    cls = enc.copy_buffer(_native.BUF_CLS, np.uint8, F * ty * tx).reshape(G, n, ty, tx)
    nr = enc.copy_buffer(_native.BUF_N_RUNS, np.int32, F * ty).reshape(G, n, ty)
    rl = enc.copy_buffer(_native.BUF_RUN_LEN, np.uint16, F * ty * tx).reshape(G, n, ty, tx)
    k = cfg.k_index
    for name, sel in (("key", [k]), ("P", [i for i in range(n) if i != k])):
        c = cls[:, sel]
        runs = nr[:, sel]
        lens = np.concatenate([rl[g, f, r, :runs[g, i, r]] for g in range(G) for i, f in enumerate(sel)
                               for r in range(ty)]) if runs.sum() else np.zeros(0)
        chains = runs.size
        tiles = c.size
        print(f"{name}: chains {chains}, tiles {tiles}, class0 {np.mean(c == 0):.3f} class1 {np.mean(c == 1):.3f} "
              f"class2 {np.mean(c == 2):.3f}; runs {runs.sum()} ({runs.sum() / chains:.1f}/chain), "
              f"mean len {lens.mean() if lens.size else 0:.2f}, max {lens.max() if lens.size else 0}, "
              f"tiles in runs {lens.sum()}")


if __name__ == "__main__":
    main()
