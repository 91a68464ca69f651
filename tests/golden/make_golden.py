"""Generate tests/golden/*.npz from the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Each fixture holds the exact inputs (float32/float64 clouds, poses), the
reference's outputs (blob bytes, project() range grid + winner indices +
counts, Huffman code lengths) and the trig tables numpy produced here, so a
test can tell an oracle bug from a host-libm difference.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import stpc  # noqa: E402  (the reference)
from stpc import huffman as ref_huffman  # noqa: E402
from stpc.motion import RigidTransform  # noqa: E402
from stpc.range_image import project as ref_project  # noqa: E402

from paper_2008_06972_b200 import synth  # noqa: E402

SMALL = synth.Sensor(360, 12, 2 * math.pi / 360, math.radians(2.2), math.radians(88.0))


def ref_cfg(sensor, n, tau, tw, th, k=None, mode=None):
    return stpc.CodecConfig(
        mode=mode or ("stream" if n > 1 else "single"), tau=tau, tile_w=tw, tile_h=th,
        res=stpc.AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
        w=sensor.w, h=sensor.h, n_frames=n, k_index=k,
    )


def save_case(name, clouds, poses, cfg, blob, extra=None):
    d = {
        "n_frames": cfg.n_frames, "k_index": cfg.k_index, "mode": cfg.mode, "tau": cfg.tau,
        "tile_w": cfg.tile_w, "tile_h": cfg.tile_h, "theta_r": cfg.res.theta_r,
        "phi_r": cfg.res.phi_r, "phi_offset": cfg.phi_offset, "w": cfg.w, "h": cfg.h,
        "range_quant": cfg.range_quant,
        "blob": np.frombuffer(blob, np.uint8),
    }
    for i, c in enumerate(clouds):
        d[f"cloud{i}"] = c
    if poses is not None:
        d["pose_R"] = np.stack([p[0] for p in poses])
        d["pose_T"] = np.stack([p[1] for p in poses])
    theta = (np.arange(cfg.w, dtype=np.float64) + 0.5) * cfg.res.theta_r
    phi = cfg.phi_offset + (np.arange(cfg.h, dtype=np.float64) + 0.5) * cfg.res.phi_r
    d["trig"] = np.concatenate([np.sin(theta), np.cos(theta), np.sin(phi), np.cos(phi)])
    d.update(extra or {})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, len(blob), "bytes blob")


def compress_case(name, seed, n, tau, tw, th, k=None, sensor=SMALL, f64=False, mutate=None, **scene):
    g = synth.make_group(seed, n, sensor, **scene)
    clouds = [c.astype(np.float64) for c in g.clouds] if f64 else list(g.clouds)
    if mutate:
        clouds = mutate(clouds)
    cfg = ref_cfg(sensor, n, tau, tw, th, k)
    poses = [RigidTransform(R=R, T=T) for R, T in g.poses] if n > 1 else None
    blob, rep = stpc.compress(clouds, cfg, poses=poses)
    # the reference's per-frame projection of the transformed clouds
    ts = stpc.poses_to_transforms(poses, cfg.k_index) if n > 1 else [RigidTransform.identity()]
    ts = [t.round_f32() for t in ts]
    extra = {}
    for i, (c, t) in enumerate(zip(clouds, ts)):
        img, win = ref_project(t.apply(c), cfg.res, cfg.w, cfg.h, cfg.phi_offset, return_indices=True)
        extra[f"ranges{i}"] = img.ranges
        extra[f"win{i}"] = win.astype(np.int32)
        extra[f"counts{i}"] = np.array([img.stats.rejected_nonfinite, img.stats.dropped_fov,
                                        img.stats.collisions], np.int64)
    extra["fractions"] = np.array([rep.fractions["temporal"], rep.fractions["spatial"], rep.fractions["residual"]])
    # the reference decoder's output, as exact-bytes digests + point counts
    dec = stpc.decompress(blob)
    extra["dec_sha256"] = np.array([hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in dec])
    extra["dec_counts"] = np.array([p.shape[0] for p in dec], np.int64)
    save_case(name, clouds, g.poses if n > 1 else None, cfg, blob, extra)


def with_bad_points(clouds):
    out = [c.copy() for c in clouds]
    c = out[0]
    c[3] = np.nan
    c[7] = 0.0
    c[11] = [0.0, 0.0, 50.0]  # straight up: outside the polar window -> dropped
    c[13] = c[12]  # exact duplicate -> collision, first index wins
    return out


def with_f64_jitter(clouds):
    """float64 clouds that are not float32-representable: the transform's
    products are inexact, so the BLAS FMA contraction shows in the bits."""
    rng = np.random.default_rng(7)
    return [c * (1.0 + rng.uniform(-1e-6, 1e-6, c.shape)) for c in clouds]


def with_empty_frame(clouds):
    out = list(clouds)
    out[0] = np.zeros((0, 3), np.float32)
    return out


def huffman_cases():
    rng = np.random.default_rng(5)
    hists = []
    hists.append(rng.integers(0, 1000, 256))
    h = np.zeros(256, np.int64); h[7] = 5; hists.append(h)  # single symbol
    h = np.zeros(256, np.int64); h[[1, 200]] = [3, 3]; hists.append(h)  # tie
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    h = np.zeros(256, np.int64); h[:40] = fib; hists.append(h)  # depth > 32 -> cap repair
    h = np.ones(256, np.int64); hists.append(h)
    h = (rng.pareto(1.2, 256) * 100).astype(np.int64); hists.append(h)
    hists = np.stack(hists)
    lens = np.stack([ref_huffman.code_lengths_from_counts(x) for x in hists])
    codes = np.stack([ref_huffman.canonical_codes(l) for l in lens])
    np.savez_compressed(os.path.join(HERE, "huffman.npz"), hists=hists, lens=lens, codes=codes)
    print("huffman", lens.max(axis=1))


def projection_cases():
    """The reference's own projection unit-test shapes (pkg/tests/test_range_image.py)."""
    out = {}
    res = stpc.AngularResolution(theta_r=np.pi / 4, phi_r=np.pi / 4)
    cases = {
        "k45": (np.array([[1.0, 1.0, np.sqrt(2.0)]]), res, 8, 4, 0.0),
        "collide": (np.array([[0.0, 2.0, 0.0], [0.0, 3.0, 0.0]]), res, 8, 4, 0.0),
        "counts": (np.array([[np.nan, 1.0, 0.0], [0.0, 0.0, 0.0], [0.0, 1.0, 5.0], [1.0, 1.0, 0.0]]),
                   stpc.AngularResolution(0.1, 0.1), 63, 4, 1.4),
        "random": (np.random.default_rng(20240811).uniform(-20, 20, (5000, 3)),
                   stpc.AngularResolution(0.02, 0.02), 315, 60, 1.0),
        "wrap": (np.array([[-1e-9, 1.0, 0.0], [1e-9, 1.0, 0.0], [-1e-300, 5.0, 0.1], [0.0, -3.0, 0.0]]),
                 stpc.AngularResolution(2 * np.pi / 360, 0.01), 360, 300, 0.0),
    }
    for name, (pts, r, w, h, off) in cases.items():
        img, win = ref_project(pts, r, w, h, off, return_indices=True)
        out[f"{name}_pts"] = pts
        out[f"{name}_geom"] = np.array([r.theta_r, r.phi_r, off, w, h])
        out[f"{name}_ranges"] = img.ranges
        out[f"{name}_win"] = win
        out[f"{name}_counts"] = np.array([img.stats.rejected_nonfinite, img.stats.dropped_fov, img.stats.collisions])
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **out)
    print("projection", list(cases))


def imu_case(name, seed, n, tau, tw, th, sensor=SMALL):
    """compress() through the IMU path (motion.py:119-207): a 200 Hz trace with
    a gap, reference frame_transforms stored as the case's poses (the key is
    identity, so poses_to_transforms on them is an exact no-op) plus the trace."""
    g = synth.make_group(seed, n, sensor)
    rng = np.random.default_rng(seed)
    t = np.round(np.arange(0.0, 0.1 * n + 0.05, 0.005), 6)
    t = np.delete(t, [40, 41, 42])  # a gap > 2x nominal (logged, not an error)
    accel = rng.normal([0.8, 0.1, 0.0], 0.3, (t.size, 3))
    gyro = rng.normal([0.0, 0.0, 0.15], 0.02, (t.size, 3))
    imu = [stpc.ImuSample(t=float(a), accel=b, gyro=c) for a, b, c in zip(t, accel, gyro)]
    frame_times = [0.013 + 0.1 * i for i in range(n)]
    v0 = np.array([9.5, 0.2, 0.0])
    cfg = ref_cfg(sensor, n, tau, tw, th, None)
    blob, rep = stpc.compress(g.clouds, cfg, imu_samples=imu, frame_times=frame_times, v0=v0)
    ts = stpc.frame_transforms(imu, frame_times, cfg.k_index, v0)
    dec = stpc.decompress(blob)
    extra = dict(fractions=np.array([rep.fractions["temporal"], rep.fractions["spatial"], rep.fractions["residual"]]),
                 imu_t=t, imu_accel=accel, imu_gyro=gyro, frame_times=np.array(frame_times), v0=v0,
                 dec_sha256=np.array([hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in dec]),
                 dec_counts=np.array([p.shape[0] for p in dec], np.int64))
    for i, (c, tr) in enumerate(zip(g.clouds, [x.round_f32() for x in ts])):
        img, win = ref_project(tr.apply(c), cfg.res, cfg.w, cfg.h, cfg.phi_offset, return_indices=True)
        extra[f"ranges{i}"] = img.ranges
        extra[f"win{i}"] = win.astype(np.int32)
        extra[f"counts{i}"] = np.array([img.stats.rejected_nonfinite, img.stats.dropped_fov,
                                        img.stats.collisions], np.int64)
    save_case(name, list(g.clouds), [(x.R, x.T) for x in ts], cfg, blob, extra)


# ----------------------------------------------------------- decoder errors


def _wrap(payload: bytes, lengths=None, encoded=None, raw_len=None, crc=None, magic=b"STPC", version=1):
    """Entropy-code a raw payload the way serialize does (bitstream.py:279-289)."""
    import struct
    import zlib

    if lengths is None:
        lengths, encoded = ref_huffman.encode_bytes(payload)
    lengths = np.asarray(lengths, np.uint8)
    raw_len = len(payload) if raw_len is None else raw_len
    crc = zlib.crc32(encoded) & 0xFFFFFFFF if crc is None else crc
    return struct.pack("<4sHHQQI", magic, version, 0, raw_len, len(encoded), crc) + lengths.tobytes() + encoded


def _varint(vals):
    out = bytearray()
    for v in vals:
        v = int(v)
        while v >= 128:
            out.append((v & 0x7F) | 0x80)
            v >>= 7
        out.append(v)
    return bytes(out)


def _layout(pl: bytes):
    """Byte positions of every section of a raw payload (bitstream.py:193-278)."""
    import struct

    (mode, tau, tw, th, tr, pr, po, w, h, n, k, q) = struct.unpack_from("<Bd HH ddd II HH d", pl, 0)
    tx, ty, nb, pm = -(-w // tw), -(-h // th), (w * h + 7) // 8, (n + 7) // 8
    L = dict(n=n, k=k, tx=tx, ty=ty, P=w * h, bits=57 + 48 * n, runs=[], fb=[], res=[])
    pos = 57 + 48 * n + n * nb
    L["nruns"] = pos
    (nr,) = struct.unpack_from("<I", pl, pos)
    pos += 4
    for _ in range(nr):
        mask = pl[pos + 18:pos + 18 + pm]
        present = [ch for ch in range(n) if mask[ch >> 3] & (1 << (ch & 7))]
        extra = len([c for c in present if c != k])
        L["runs"].append(dict(pos=pos, extra=extra, present=present))
        pos += 18 + pm + 4 * extra
    for ch in range(n):
        pc = pos
        (nrows,) = struct.unpack_from("<I", pl, pos)
        pos += 4
        rows = []
        for _ in range(nrows):
            row, nrr = struct.unpack_from("<HH", pl, pos)
            rows.append(dict(pos=pos, nr=nrr, runs=pos + 4))
            pos += 4 + 16 * nrr
        L["fb"].append(dict(pos=pc, rows=rows))
    for ch in range(n):
        pc = pos
        (cnt,) = struct.unpack_from("<I", pl, pos)
        pos += 4
        if cnt == 0:
            L["res"].append(dict(pos=pc, cnt=0))
            continue
        var = pos
        vals = []
        for _ in range(cnt):
            v = sh = 0
            while True:
                b = pl[pos]
                pos += 1
                v |= (b & 0x7F) << sh
                if b < 128:
                    break
                sh += 7
            vals.append(v)
        code = pos
        pos += 2 * cnt
        (ne,) = struct.unpack_from("<I", pl, pos)
        L["res"].append(dict(pos=pc, cnt=cnt, var=var, deltas=vals, code=code, nesc=pos, esc=pos + 4, n_esc=ne))
        pos += 4 + 4 * ne
    L["end"] = pos
    assert pos == len(pl)
    return L


def decode_error_cases():
    """Corrupted blobs and the exception the reference's decompress raises for
    each (tests/test_gpu_parity.py::test_decode_errors_match_reference)."""
    import struct

    g = synth.make_group(301, 3, SMALL)
    import dataclasses

    cfg = dataclasses.replace(ref_cfg(SMALL, 3, 0.1, 4, 4), range_quant=0.0003)  # ranges > 19.7 m escape
    poses = [RigidTransform(R=R, T=T) for R, T in g.poses]
    blob, _ = stpc.compress(g.clouds, cfg, poses=poses)
    enc, _ = stpc.bitstream.deserialize(blob)
    raw_len, enc_len = struct.unpack_from("<QQ", blob, 8)
    pl = stpc.huffman.decode_bytes(np.frombuffer(blob, np.uint8, 256, 28), blob[284:284 + enc_len], raw_len)
    L = _layout(pl)
    n, k, tx, ty, P = L["n"], L["k"], L["tx"], L["ty"], L["P"]
    run_x = next(r for r in L["runs"] if r["extra"] > 0)
    fb_ch = next(c for c in range(n) if L["fb"][c]["rows"])
    fb_row = L["fb"][fb_ch]["rows"][0]
    res_ch = next(c for c in range(n) if L["res"][c]["cnt"] > 3 and L["res"][c]["n_esc"] > 0)
    R = L["res"][res_ch]
    print("layout: runs", len(L["runs"]), "fb rows", sum(len(f["rows"]) for f in L["fb"]),
          "res", [r["cnt"] for r in L["res"]], "esc", [r.get("n_esc", 0) for r in L["res"]])

    def put(b, off, fmt, *v):
        b = bytearray(b)
        struct.pack_into(fmt, b, off, *v)
        return bytes(b)

    def one_byte_delta(r):
        # index i > 0 of a one-byte varint
        pos = r["var"]
        for i, d in enumerate(r["deltas"]):
            ln = len(_varint([d]))
            if i > 0 and ln == 1:
                return pos
            pos += ln
        raise AssertionError

    def with_deltas(b, r, deltas):
        return b[:r["var"]] + _varint(deltas) + b[r["code"]:]

    pcases = {
        "ok": pl,
        "trunc_config": pl[:30],
        "trunc_transforms": pl[:57 + 10],
        "trunc_bitmaps": pl[:L["bits"] + 5],
        "trunc_nruns": pl[:L["nruns"] + 2],
        "trunc_run_header": pl[:run_x["pos"] + 10],
        "trunc_run_mask": pl[:run_x["pos"] + 18],
        "trunc_run_offsets": pl[:run_x["pos"] + 19 + 2],
        "trunc_fb_count": pl[:L["fb"][0]["pos"] + 2],
        "trunc_fb_row": pl[:fb_row["pos"] + 2],
        "trunc_fb_runs": pl[:fb_row["runs"] + 8],
        "trunc_res_count": pl[:L["res"][0]["pos"] + 3],
        "trunc_varints": pl[:R["var"] + 2],
        "trunc_codes": pl[:R["code"] + 3],
        "trunc_nesc": pl[:R["nesc"] + 1],
        "trunc_escapes": pl[:R["esc"] + 2],
        "trailing_bytes": pl + b"\x00\x00",
        "cfg_mode": put(pl, 0, "<B", 7),
        "cfg_tau_neg": put(pl, 1, "<d", -1.0),
        "cfg_tau_nan": put(pl, 1, "<d", float("nan")),
        "cfg_tile0": put(pl, 9, "<H", 0),
        "cfg_frames0": put(pl, 45, "<H", 0),
        "cfg_k_oob": put(pl, 47, "<H", n),
        "cfg_single_multi": put(pl, 0, "<B", 0),
        "cfg_huge_image": put(pl, 37, "<II", 70000, 1000),
        "xf_not_orthonormal": put(pl, 57 + 48, "<f", 2.0),
        "xf_nan": put(pl, 57 + 48 + 36, "<f", float("nan")),
        "run_row_oob": put(pl, run_x["pos"], "<H", ty),
        "run_len0": put(pl, run_x["pos"] + 4, "<H", 0),
        "run_span_oob": put(pl, run_x["pos"] + 2, "<H", tx - 1),
        "run_no_key": put(pl, run_x["pos"] + 18, "<B", pl[run_x["pos"] + 18] & ~(1 << k)),
        "fb_nrows_oob": put(pl, L["fb"][fb_ch]["pos"], "<I", ty + 1),
        "fb_row_oob": put(pl, fb_row["pos"], "<H", ty),
        "fb_nr_oob": put(pl, fb_row["pos"] + 2, "<H", tx + 1),
        "fb_run_len0": put(pl, fb_row["runs"] + 2, "<H", 0),
        "fb_run_span_oob": put(pl, fb_row["runs"], "<H", tx),
        "res_count_oob": put(pl, R["pos"], "<I", P + 1),
        "res_delta_zero": put(pl, one_byte_delta(R), "<B", 0),
        "res_overlong_varint": pl[:R["var"]] + b"\x80" * 11 + pl[R["var"] + 11:],
        "res_flat_oob": with_deltas(pl, R, [R["deltas"][0] + P] + R["deltas"][1:]),
        "res_delta_too_big": with_deltas(pl, R, R["deltas"][:1] + [P + 1] + R["deltas"][2:]),
        "res_escape_mismatch": put(pl, R["nesc"], "<I", R["n_esc"] - 1)[:R["esc"] + 4 * (R["n_esc"] - 1)]
        + pl[R["esc"] + 4 * R["n_esc"]:],
        # two errors: the reference reports the first in reading order
        "two_run_len0_then_trunc": put(pl, run_x["pos"] + 4, "<H", 0)[:R["code"] + 1],
        "two_row_oob_mask_trunc": put(pl, run_x["pos"], "<H", ty)[:run_x["pos"] + 18],
        "two_delta_zero_then_trunc_codes": put(pl, one_byte_delta(R), "<B", 0)[:R["code"] + 3],
        "two_fb_oob_then_trailing": put(pl, fb_row["pos"], "<H", ty) + b"\x01",
        "two_no_key_then_res_oob": put(put(pl, run_x["pos"] + 18, "<B", pl[run_x["pos"] + 18] & ~(1 << k)),
                                       R["pos"], "<I", P + 1),
    }
    blobs = {name: _wrap(b) for name, b in pcases.items()}
    # header / code table / entropy-stage cases
    lens, encd = ref_huffman.encode_bytes(pl)
    blobs["hdr_short"] = blob[:100]
    blobs["hdr_magic"] = b"XTPC" + blob[4:]
    blobs["hdr_version"] = blob[:4] + b"\x02\x00" + blob[6:]
    blobs["hdr_raw_cap"] = put(blob, 8, "<Q", (1 << 30) + 1)
    blobs["hdr_enc_past_end"] = blob[:-10]
    blobs["hdr_crc"] = put(blob, 24, "<I", (struct.unpack_from("<I", blob, 24)[0] ^ 1))
    bad = np.array(lens, np.uint8)
    bad[np.flatnonzero(bad)[0]] = 33
    blobs["table_len33"] = _wrap(pl, bad, encd)
    blobs["table_overflow"] = _wrap(pl, np.ones(256, np.uint8), encd)
    blobs["table_empty"] = _wrap(pl, np.zeros(256, np.uint8), encd)
    blobs["raw_len0"] = _wrap(b"", np.zeros(256, np.uint8), b"", raw_len=0)
    one = np.zeros(256, np.uint8)
    one[65] = 1
    blobs["huff_invalid_code"] = _wrap(b"", one, b"\x00\xff\xff\xff\xff\xff\xff\xff", raw_len=20)
    blobs["huff_invalid_after_end"] = _wrap(b"", one, b"\x00\x00\xff\xff\xff\xff\xff\xff", raw_len=16)
    blobs["huff_truncated"] = _wrap(b"", one, b"\x00\x00", raw_len=40)
    blobs["huff_short_tail"] = _wrap(b"", one, b"\x00\x00\xff\xff", raw_len=20)
    names, expect, data = [], [], []
    for name, b in blobs.items():
        try:
            stpc.decompress(b)
            exc = "ok"
        except Exception as e:  # noqa: BLE001
            exc = type(e).__name__
        names.append(name)
        expect.append(exc)
        data.append(np.frombuffer(b, np.uint8))
        print(f"  {name:34s} {exc}")
    off = np.zeros(len(data) + 1, np.int64)
    off[1:] = np.cumsum([d.size for d in data])
    np.savez_compressed(os.path.join(HERE, "decode_errors.npz"), names=np.array(names), expect=np.array(expect),
                        blobs=np.concatenate(data), offsets=off)


def overlap_cases():
    """Blobs whose runs overlap or come out of order -- the encoder never
    writes them, but the reference's deserialize accepts them and its decoder
    applies temporal runs, then fallback runs, in stream order: per pixel the
    last successful reconstruction wins and each failed (run, pixel) counts
    (temporal.py:307-331, _kernels.py:282-308).  Built by editing a real
    StreamEncoded and re-serializing it with the reference's own serialize;
    the expected decode is the reference's decompress_full."""
    import dataclasses

    from stpc.bitstream import decompress_full, deserialize, serialize
    from stpc.plane import Plane
    from stpc.spatial import EncodedRow, PlaneRun

    g = synth.make_group(311, 4, SMALL, n_boxes=25)
    cfg = ref_cfg(SMALL, 4, 0.1, 4, 4)
    poses = [RigidTransform(R=R, T=T) for R, T in g.poses]
    blob, _ = stpc.compress(g.clouds, cfg, poses=poses)
    enc, cfg2 = deserialize(blob)
    k = enc.k_index
    tr = enc.temporal_runs
    long_i = max(range(len(tr)), key=lambda i: tr[i].length)
    lr = tr[long_i]
    out = {}

    def shifted(run, ds, dlen, da=0.0, dc=0.0, offsets=None):
        pl = Plane(float(np.float32(run.plane.a + da)), float(np.float32(run.plane.b)),
                   float(np.float32(run.plane.c + dc)))
        offs = offsets if offsets is not None else [
            None if o is None else float(np.float32(o + dc)) for o in run.offsets]
        return dataclasses.replace(run, s=run.s + ds, length=run.length + dlen, plane=pl, offsets=offs)

    # (1) a temporal run overlapping the longest one, later in the stream,
    #     with a tilted plane; every channel present
    extra = shifted(lr, max(0, lr.length // 3), -(lr.length // 3) if lr.length > 2 else 0, da=0.02, dc=0.3,
                    offsets=[float(np.float32(o + 0.3)) if o is not None else float(np.float32(lr.plane.c + 0.1))
                             for o in lr.offsets])
    out["t_overlap"] = dataclasses.replace(enc, temporal_runs=tr + [extra])
    # (2) the same overlap with a negative offset on one channel: r_hat <= 0
    #     fails there, so the earlier run's value must survive
    bad = dataclasses.replace(extra, offsets=[(-5.0 if ch == (k + 1) % enc.n else o)
                                              for ch, o in enumerate(extra.offsets)])
    out["t_overlap_fail"] = dataclasses.replace(enc, temporal_runs=tr + [bad])
    # (3) temporal runs in reverse stream order (disjoint): decodes as (0)
    out["t_reversed"] = dataclasses.replace(enc, temporal_runs=list(reversed(tr)))
    # (4) fallback: a duplicated row with another plane, plus an overlapping
    #     run inside a row
    ch = max((c for c in range(enc.n) if c != k), key=lambda c: len(enc.fallback_rows[c]))
    rows = list(enc.fallback_rows[ch])
    assert len(rows) >= 3
    r0 = rows[0]
    run0 = r0.runs[0]
    ov = PlaneRun(s=run0.s, length=run0.length, plane=Plane(float(np.float32(run0.plane.a)),
                  float(np.float32(run0.plane.b + 0.01)), float(np.float32(run0.plane.c + 0.2))))
    dup = EncodedRow(row_id=r0.row_id, runs=[ov])
    inner = EncodedRow(row_id=rows[-2].row_id, runs=list(rows[-2].runs) + [
        PlaneRun(s=rows[-2].runs[0].s, length=1, plane=Plane(0.0, 0.0, -1.0))])  # r_hat < 0: failures
    fb = [list(x) for x in enc.fallback_rows]
    fb[ch] = rows[:-2] + [inner, dup]  # same row count (the format caps it at tiles_y)
    out["fb_overlap"] = dataclasses.replace(enc, fallback_rows=fb)

    names, data, shas, counts, failed = [], [], [], [], []
    for name, e in out.items():
        b = serialize(e, cfg2)
        clouds, rep = decompress_full(b)
        names.append(name)
        data.append(np.frombuffer(b, np.uint8))
        shas.append([hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in clouds])
        counts.append([p.shape[0] for p in clouds])
        failed.append(rep.failed_reconstructions)
        print(f"  {name:16s} {len(b)} B, failed {rep.failed_reconstructions}, points {counts[-1]}")
    off = np.zeros(len(data) + 1, np.int64)
    off[1:] = np.cumsum([d.size for d in data])
    theta = (np.arange(SMALL.w, dtype=np.float64) + 0.5) * SMALL.theta_r
    phi = SMALL.phi_offset + (np.arange(SMALL.h, dtype=np.float64) + 0.5) * SMALL.phi_r
    np.savez_compressed(os.path.join(HERE, "decode_overlap.npz"), names=np.array(names), blobs=np.concatenate(data),
                        offsets=off, dec_sha256=np.array(shas), dec_counts=np.array(counts),
                        failed=np.array(failed, np.int64),
                        trig=np.concatenate([np.sin(theta), np.cos(theta), np.sin(phi), np.cos(phi)]))


CASES = {
    "single_4x4": lambda: compress_case("single_4x4", 101, 1, 0.1, 4, 4),
    "stream3_4x4": lambda: compress_case("stream3_4x4", 102, 3, 0.1, 4, 4),
    "stream5_2x2": lambda: compress_case("stream5_2x2", 103, 5, 0.2, 2, 2),
    "stream4_8x4_k0": lambda: compress_case("stream4_8x4_k0", 104, 4, 0.05, 8, 5, k=0),
    "single_f64_bad": lambda: compress_case("single_f64_bad", 105, 1, 0.1, 4, 4, f64=True, mutate=with_bad_points),
    "stream3_empty": lambda: compress_case("stream3_empty", 106, 3, 0.1, 4, 4, mutate=with_empty_frame),
    "stream6_16x16": lambda: compress_case("stream6_16x16", 107, 6, 0.02, 16, 16),
    "stream5_imu": lambda: imu_case("stream5_imu", 109, 5, 0.1, 4, 4),
    "stream4_f64": lambda: compress_case("stream4_f64", 108, 4, 0.1, 4, 4, f64=True, mutate=with_f64_jitter),
}

if __name__ == "__main__":
    # python tests/golden/make_golden.py [case ...]   (no args: everything)
    only = sys.argv[1:]
    if not only:
        projection_cases()
        huffman_cases()
    if not only or "decode_errors" in only:
        decode_error_cases()
    if not only or "decode_overlap" in only:
        overlap_cases()
    for name, fn in CASES.items():
        if not only or name in only:
            fn()
