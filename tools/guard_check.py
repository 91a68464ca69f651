"""Out-of-bounds write check of every kernel (the pool has no compute-sanitizer).

Runs the encoder and decoder over small and odd workloads with the
write-guard build libstpc_b200_guard.so (-DSTPC_GUARD: the bytes past each
workspace's requested size hold a canary) and checks the canaries after every
call; the blobs are also compared with the oracle.  A kernel writing past the
end of any of its buffers makes a check fail.  Also repeats each encode and
requires identical bytes (a shared-memory or work-stealing race would show as
run-to-run differences).

    python tools/guard_check.py [--out gpurun_out/guard.json]
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["STPC_B200_LIB"] = os.path.join(ROOT, "paper_2008_06972_b200", "libstpc_b200_guard.so")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from conftest import GOLDEN, golden_cases, load_case  # noqa: E402
from oracle import decode as odec  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2008_06972_b200 import (  # noqa: E402
    AngularResolution, CodecConfig, Encoder, _native, compress, compress_groups, decompress, decompress_full,
    decompress_many, release_cached, synth)
from paper_2008_06972_b200.geometry import poses_to_transforms  # noqa: E402

L = _native.load(require_device=True)
L.stpc_debug_guard_check.argtypes = [ctypes.c_char_p, ctypes.c_int32]
L.stpc_debug_guard_check.restype = ctypes.c_int64
L.stpc_debug_guard_buffers.restype = ctypes.c_int32

LOG = {"checks": 0, "buffers_max": 0, "cases": {}, "violations": []}


def guard(case):
    buf = ctypes.create_string_buffer(8192)
    bad = L.stpc_debug_guard_check(buf, 8192)
    LOG["checks"] += 1
    LOG["buffers_max"] = max(LOG["buffers_max"], L.stpc_debug_guard_buffers())
    if bad != 0:
        LOG["violations"].append({"case": case, "bytes": int(bad), "report": buf.value.decode()})
        print(f"GUARD VIOLATION in {case}: {bad}\n{buf.value.decode()}", flush=True)


def record(case, ok):
    LOG["cases"][case] = bool(ok)
    if not ok:
        print(f"MISMATCH in {case}", flush=True)


def fuzz(seeds):
    for seed in seeds:
        rng = np.random.default_rng(9000 + seed)
        w, h = int(rng.integers(8, 400)), int(rng.integers(2, 40))
        wide = seed % 5 == 0  # sensor narrower than the full circle: the azimuth wraps
        tr = (2 * np.pi / 1800 if wide else 2 * np.pi / w * float(rng.uniform(0.5, 1.0)))
        sensor = synth.Sensor(w, h, tr, float(rng.uniform(0.01, 0.06)), float(rng.uniform(1.2, 1.7)))
        n = int(rng.integers(1, 10))
        tw, th = int(rng.integers(1, 9)), int(rng.integers(1, 7))
        grp = synth.make_group(9100 + seed, n, sensor, n_boxes=int(rng.integers(2, 30)),
                               noise=float(rng.uniform(0.0, 0.05)), dropout=float(rng.uniform(0.0, 0.5)))
        clouds = list(grp.clouds)
        if seed % 4 == 3:
            clouds = [c.astype(np.float64) * (1.0 + 1e-7) for c in clouds]
        if seed % 7 == 2 and n > 1:
            clouds[0] = np.zeros((0, 3), clouds[0].dtype)
        cfg = CodecConfig(mode="single" if n == 1 else "stream", tau=float(rng.choice([0.005, 0.05, 0.3, 1.0])),
                          tile_w=tw, tile_h=th, res=AngularResolution(sensor.theta_r, sensor.phi_r),
                          phi_offset=sensor.phi_offset, w=w, h=h, n_frames=n,
                          k_index=None if n == 1 else int(rng.integers(0, n)),
                          range_quant=float(rng.choice([0.0005, 0.005, 0.05])))
        poses = grp.poses if n > 1 else None
        a, _ = compress(clouds, cfg, poses=poses)
        guard(f"fuzz{seed}/encode")
        b, _ = compress(clouds, cfg, poses=poses)
        ref, _ = oracle.compress(clouds, cfg, poses)
        mine = decompress(a)
        guard(f"fuzz{seed}/decode")
        ok = a == b == ref and all(np.array_equal(x, y) for x, y in zip(mine, odec.decompress(a)))
        record(f"fuzz{seed}", ok)


def goldens():
    for name in golden_cases():
        clouds, poses, cfg, blob, z = load_case(name)
        mine, _ = compress(clouds, cfg, poses=poses)
        guard(f"golden/{name}/encode")
        out = decompress(blob)
        guard(f"golden/{name}/decode")
        record(f"golden/{name}", mine == oracle.compress(clouds, cfg, poses)[0] and
               all(np.array_equal(x, y) for x, y in zip(out, odec.decompress(blob))))


def corrupt_and_overlap():
    z = np.load(os.path.join(GOLDEN, "decode_errors.npz"))
    got = []
    for i, (name, expect) in enumerate(zip(z["names"], z["expect"])):
        blob = z["blobs"][z["offsets"][i]:z["offsets"][i + 1]].tobytes()
        try:
            decompress(blob)
            exc = "ok"
        except Exception as e:  # noqa: BLE001
            exc = type(e).__name__
        guard(f"corrupt/{name}")
        got.append(exc == str(expect))
    record("corrupt_blobs", all(got))
    z = np.load(os.path.join(GOLDEN, "decode_overlap.npz"))
    ok = True
    for i, name in enumerate(z["names"]):
        blob = z["blobs"][z["offsets"][i]:z["offsets"][i + 1]].tobytes()
        clouds, rep = decompress_full(blob)
        guard(f"overlap/{name}")
        ref, failed = odec.decompress_full(blob)
        ok &= rep.failed_reconstructions == failed and all(np.array_equal(a, b) for a, b in zip(clouds, ref))
    record("overlap_blobs", ok)


def batches():
    sensor = synth.Sensor(300, 12, 2 * math.pi / 300, math.radians(2.0), math.radians(88.0))
    cfg = CodecConfig(mode="stream", tau=0.1, tile_w=4, tile_h=3, res=AngularResolution(sensor.theta_r, sensor.phi_r),
                      phi_offset=sensor.phi_offset, w=sensor.w, h=sensor.h, n_frames=3)
    groups, poses = [], []
    for gi in range(131):
        grp = synth.make_group(8000 + gi, 3, sensor, n_boxes=4)
        clouds = list(grp.clouds)
        if gi % 17 == 5:
            clouds[1] = np.zeros((0, 3), np.float32)
        groups.append(clouds)
        poses.append(grp.poses)
    blobs, _ = compress_groups(groups, cfg, poses)  # gather pipeline, 16 chunks
    guard("compress_groups/131")
    again, _ = compress_groups(groups, cfg, poses)
    ok = blobs == again and all(blobs[g] == oracle.compress(groups[g], cfg, poses[g])[0] for g in (0, 5, 64, 130))
    clouds, _ = decompress_many(blobs)
    guard("decompress_many/131")
    record("compress_groups_131", ok)
    # pipelined host encode from one buffer + one-shot
    enc = Encoder(cfg)
    pts = np.ascontiguousarray(np.concatenate([c for grp in groups for c in grp]))
    off = np.zeros(3 * 131 + 1, np.int64)
    off[1:] = np.cumsum([c.shape[0] for grp in groups for c in grp])
    xf = np.asarray([t.round_f32().row12() for p in poses for t in poses_to_transforms(p, 1)])
    enc.encode_host(131, pts, off, xf)
    guard("encode_host/one_shot")
    one = enc.blobs()
    out = np.zeros(sum(len(b) + 16 for b in one) + 4096, np.uint8)
    enc.encode_host(131, pts, off, xf, out)
    guard("encode_host/pipelined")
    o, ln = enc.blob_layout()
    record("encode_host_pipelined", [out[a:a + m].tobytes() for a, m in zip(o[:-1], ln)] == one == blobs)
    del enc


def headline_batch(G=64):
    import torch

    sensor, n, tile, tau, scene = synth.config_params(4)
    cfg = CodecConfig(mode="stream", tau=tau, tile_w=tile, tile_h=tile,
                      res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                      w=sensor.w, h=sensor.h, n_frames=n)
    frames, xf, groups, poses = [], [], [], []
    for g in range(G):
        grp = synth.make_group(1_000_003 * 4 + g, n, sensor, device="cuda", as_numpy=False, **scene)
        frames.extend(grp.clouds)
        xf.extend(t.round_f32().row12() for t in poses_to_transforms(grp.poses, n // 2))
        groups.append([c.cpu().numpy() for c in grp.clouds])
        poses.append(grp.poses)
    d = torch.cat(frames).contiguous()
    off = np.zeros(len(frames) + 1, np.int64)
    off[1:] = np.cumsum([f.shape[0] for f in frames])
    enc = Encoder(cfg)
    enc.encode_device(G, d.data_ptr(), off, np.asarray(xf))
    guard(f"encode_device/{G}x8")
    blobs = enc.blobs()
    enc.encode_device(G, d.data_ptr(), off, np.asarray(xf))
    guard(f"encode_device/{G}x8/again")
    ok = enc.blobs() == blobs and all(blobs[g] == oracle.compress(groups[g], cfg, poses[g])[0] for g in (0, G - 1))
    decompress_many(blobs)
    guard(f"decompress_many/{G}x8")
    record(f"encode_device_{G}", ok)


def entropy_and_project():
    fib = [1, 1]
    while len(fib) < 36:
        fib.append(fib[-1] + fib[-2])
    rng = np.random.default_rng(3)
    h = np.zeros(256, np.int64)
    h[:34] = fib[:34]
    p = np.repeat(np.arange(256, dtype=np.uint8), h)
    rng.shuffle(p)
    payloads = [p.tobytes(), bytes(rng.integers(0, 256, 777, dtype=np.uint8)), b"\x05" * 17]
    buf = np.frombuffer(b"".join(payloads), np.uint8)
    off = np.zeros(4, np.int64)
    off[1:] = np.cumsum([len(x) for x in payloads])
    out = np.zeros(len(buf) + 8192, np.uint8)
    oo = np.zeros(4, np.int64)
    _native.check(L.stpc_entropy_encode(buf.ctypes.data, off.ctypes.data, 3, out.ctypes.data, out.nbytes,
                                        oo.ctypes.data))
    guard("entropy_encode")
    record("entropy_encode", all(out[oo[i]:oo[i + 1]].tobytes() == oracle.entropy_blob(x)
                                 for i, x in enumerate(payloads)))


def main():
    t0 = time.time()
    fuzz(range(int(os.environ.get("STPC_GUARD_SEEDS", "40"))))
    goldens()
    corrupt_and_overlap()
    batches()
    entropy_and_project()
    headline_batch()
    release_cached()
    LOG["seconds"] = round(time.time() - t0, 1)
    LOG["all_identical"] = all(LOG["cases"].values())
    LOG["violations_total"] = len(LOG["violations"])
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    s = json.dumps(LOG, indent=1)
    if out:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        open(out, "w").write(s)
    print(json.dumps({k: LOG[k] for k in ("checks", "buffers_max", "violations_total", "all_identical", "seconds")}))
    sys.exit(1 if LOG["violations"] or not LOG["all_identical"] else 0)


if __name__ == "__main__":
    main()
