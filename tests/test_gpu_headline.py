"""Parity of the exact workload the headline number is measured on.

BASELINE.json configs[3] as bench.py runs it: 1024 seeded 64-beam groups of
1 K + 7 P frames (4x4 tiles, tau 0.1 m), encoded in ONE device pass
(stpc_encode_device: 8.4 GB range grid, work-stealing fit blocks) and through
the 24-chunk pipelined host path (stpc_encode_host).  Every one of the 1024
blobs must equal the oracle's byte for byte -- each group's blob is a pure
function of its input (/root/reference/pkg/src/stpc/bitstream.py:527-602;
/root/reference/pkg/README.md:119-120) -- and the GPU decoder must invert a
sample exactly like the oracle decoder."""

import argparse

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_headline_batch_all_groups_identical():
    import torch

    import bench
    from paper_2008_06972_b200 import Encoder

    args = argparse.Namespace(config=4, groups=None, tile=None, tau=None)
    sensor, n, tile, tau, scene, G = bench.workload(args)
    assert G == 1024 and n == 8
    cfg = bench.codec_config(sensor, n, tile, tau)
    dev = torch.device("cuda", 0)
    d_pts, off, xf = bench.make_inputs(args, 0, dev)
    enc = Encoder(cfg)
    enc.encode_device(G, d_pts.data_ptr(), off, xf)
    dev_blobs = enc.blobs()
    stats = enc.frame_stats()
    hp = d_pts.cpu().numpy()
    del d_pts
    torch.cuda.empty_cache()
    out = np.empty(sum(len(b) + 16 for b in dev_blobs) + (1 << 20), np.uint8)
    enc.encode_host(G, hp, off, xf, out)  # pipelined: 24 chunks of 43 groups
    o, ln = enc.blob_layout()
    host_blobs = [out[a:a + m].tobytes() for a, m in zip(o[:-1], ln)]
    assert host_blobs == dev_blobs
    assert np.array_equal(enc.frame_stats(), stats)

    sel = list(range(G))
    par = bench.headline_parity(cfg, n, hp, off, xf, sel, {"encode_device": dev_blobs}, decode_blobs=False)
    assert par["encode_device"]["identical"] == G, par
    # decoder on the parity sample of the bench line
    psel = bench.parity_groups(G)
    par = bench.headline_parity(cfg, n, hp, off, xf, psel, {"encode_host": [host_blobs[g] for g in psel]})
    assert par["identical"] == len(psel) and par["decode_identical"] == len(psel), par
    # every frame's valid pixels partition into temporal + fallback + residual
    assert np.array_equal(stats[:, 4] + stats[:, 5] + stats[:, 6], stats[:, 3])
