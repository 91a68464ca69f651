"""Where one decompress(blob) call spends its time (diagnostic): the kernel
launch list of one call on a BASELINE config (run under ncu for per-kernel
times) and the host wall time per phase.

    python tools/decompress_latency.py [config 1-5]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2008_06972_b200 import compress, decompress, synth  # noqa: E402
from paper_2008_06972_b200 import decode as D  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    sensor, n, tile, tau, scene = synth.config_params(cfg_id)
    cfg = bench.codec_config(sensor, n, tile, tau)
    g = synth.make_group(bench.group_seed(0, 0, cfg_id), n, sensor, device="cuda", **scene)
    blob, _ = compress(g.clouds, cfg, poses=g.poses if n > 1 else None)
    for _ in range(3):
        decompress(blob)
    ts = []
    for _ in range(10):
        t = time.perf_counter()
        clouds = decompress(blob)
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"config {cfg_id}: blob {len(blob)} B, {sum(c.shape[0] for c in clouds)} points, "
          f"decompress {sorted(ts)[len(ts) // 2]:.2f} ms")
    dec = D.get_decoder()
    t = time.perf_counter()
    _, reps, _ = dec.decode(0, None, False, host_blobs=[blob])
    print(f"timings {reps[0].timings}, total {1e3 * (time.perf_counter() - t):.2f} ms")


if __name__ == "__main__":
    main()
