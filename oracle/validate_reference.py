"""Validate the CPU oracle against the LIVE reference package (build container
only -- /root/reference is not on the GPU box).

    NUMBA_CACHE_DIR=/tmp/nb python oracle/validate_reference.py

For BASELINE-shaped groups it checks that the oracle's
compress blob is byte-identical to stpc.compress, and that the oracle
decoder's output is bit-identical to stpc.decompress.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path = [p for p in sys.path if os.path.abspath(p or ".") != os.path.dirname(os.path.abspath(__file__))]
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import stpc  # noqa: E402  (the reference)
from stpc.motion import RigidTransform  # noqa: E402

from oracle import decode as odec  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2008_06972_b200 import synth  # noqa: E402


def main():
    oracle.build()
    cases = [(1, 10, synth.SENSOR_64, 4, 0.1), (2, 1, synth.SENSOR_64, 4, 0.1), (3, 8, synth.SENSOR_64, 4, 0.1),
             (4, 5, synth.SENSOR_128, 2, 0.2), (5, 5, synth.SENSOR_128, 16, 0.02)]
    for seed, n, s, tile, tau in cases:
        g = synth.make_group(seed, n, s)
        cfg = stpc.CodecConfig(mode="stream" if n > 1 else "single", tau=tau, tile_w=tile, tile_h=tile,
                               res=stpc.AngularResolution(s.theta_r, s.phi_r), phi_offset=s.phi_offset,
                               w=s.w, h=s.h, n_frames=n)
        poses = [RigidTransform(R=R, T=T) for R, T in g.poses] if n > 1 else None
        blob, _ = stpc.compress(g.clouds, cfg, poses=poses)
        t = time.time()
        ob, _ = oracle.compress(g.clouds, cfg, g.poses if n > 1 else None)
        dt = time.time() - t
        ref_dec = stpc.decompress(blob)
        my_dec = odec.decompress(blob)
        same_dec = all(np.array_equal(a, b) for a, b in zip(ref_dec, my_dec))
        print(f"seed {seed} n {n} {s.h}b tile {tile} tau {tau}: blob {len(blob)} B identical={blob == ob} "
              f"decode identical={same_dec} (oracle {dt:.2f}s)")
        assert blob == ob and same_dec


if __name__ == "__main__":
    main()
