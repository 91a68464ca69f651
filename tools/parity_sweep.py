"""Full-size parity sweep over every BASELINE.json config (GPU; evidence for
profiles/): for each case one seeded group goes through the GPU `compress`
and through the oracle (test infrastructure), and the blobs must be
byte-identical; the GPU blob must also decode, through the GPU `decompress`,
to the oracle decoder's clouds bit for bit.

    python tools/parity_sweep.py [out.json]

Cases: configs[0], [1], [4] at full size; all 16 tile x threshold points of
configs[2]; 4 groups of configs[3] in one compress_groups call.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import decode as odec  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2008_06972_b200 import (AngularResolution, CodecConfig, compress, compress_groups,  # noqa: E402
                                   decompress, synth)


def cfg_of(sensor, n, tau, tile):
    return CodecConfig(mode="stream" if n > 1 else "single", tau=tau, tile_w=tile, tile_h=tile,
                       res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                       w=sensor.w, h=sensor.h, n_frames=n)


def same_clouds(a, b):
    return len(a) == len(b) and all(x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))
                                    for x, y in zip(a, b))


def one(name, seed, cfg_id, tile=None, tau=None):
    sensor, n, t0, tau0, scene = synth.config_params(cfg_id)
    tile, tau = tile or t0, tau or tau0
    g = synth.make_group(seed, n, sensor, device="cuda", **scene)
    cfg = cfg_of(sensor, n, tau, tile)
    poses = g.poses if n > 1 else None
    t = time.perf_counter()
    mine, rep = compress(g.clouds, cfg, poses=poses)
    t_gpu = time.perf_counter() - t
    t = time.perf_counter()
    ref, _ = oracle.compress(g.clouds, cfg, poses)
    t_cpu = time.perf_counter() - t
    row = {"case": name, "tile": tile, "tau": tau, "frames": n, "points": int(sum(c.shape[0] for c in g.clouds)),
           "blob_bytes": len(mine), "blob_identical": mine == ref, "eps_band_points": rep.eps_band_points,
           "fractions": {k: round(v, 4) for k, v in rep.fractions.items()},
           "gpu_compress_s": round(t_gpu, 4), "oracle_compress_s": round(t_cpu, 3)}
    row["decode_identical"] = same_clouds(decompress(mine), odec.decompress(ref))
    return row


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    rows = [one("configs[0] single 64b", 101, 1), one("configs[1] 1K+9P 64b", 102, 2),
            one("configs[4] single 256b dense", 105, 5)]
    for tile in (2, 4, 8, 16):
        for tau in (0.02, 0.05, 0.1, 0.2):
            rows.append(one(f"configs[2] 128b 1K+4P tile {tile} tau {tau}", 3000 + 10 * tile + int(100 * tau), 3,
                            tile, tau))
    # configs[3]: groups in one batched device pass
    sensor, n, tile, tau, scene = synth.config_params(4)
    cfg = cfg_of(sensor, n, tau, tile)
    groups = [synth.make_group(104_000 + i, n, sensor, device="cuda", **scene) for i in range(4)]
    blobs, _ = compress_groups([g.clouds for g in groups], cfg, [g.poses for g in groups])
    ok = all(b == oracle.compress(g.clouds, cfg, g.poses)[0] for g, b in zip(groups, blobs))
    rows.append({"case": "configs[3] 4 groups x 1K+7P 64b, one compress_groups call", "blob_identical": ok,
                 "frames": 4 * n})
    bad = [r["case"] for r in rows if not r["blob_identical"] or not r.get("decode_identical", True)]
    summary = {"cases": len(rows), "all_identical": not bad, "failures": bad, "rows": rows}
    text = json.dumps(summary, indent=1)
    if out:
        open(out, "w").write(text)
    print(f"parity sweep: {len(rows) - len(bad)}/{len(rows)} cases byte-identical (blobs and decodes)")


if __name__ == "__main__":
    main()
