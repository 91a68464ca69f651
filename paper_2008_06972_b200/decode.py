"""Drop-in ``decompress`` / ``decompress_full``.

Mirrors /root/reference/pkg/src/stpc/bitstream.py:605-631 (and the checks of
``deserialize`` :388-519) with the heavy work on the GPU (libstpc_b200):
CRC-32 and Huffman decoding of the entropy payload, plane reconstruction of
every pixel, residual scatter, unprojection and the inverse frame transform.
The host parses the record sections (O(runs + rows), vectorised numpy for
the residual varints) into per-tile plane maps.  ``decompress_many`` decodes
a batch of blobs that share one configuration in one device pass.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import _native
from .errors import ChecksumError, MalformedBlobError, TruncatedBlobError, UnknownVersionError
from .geometry import DEFAULT_R_MAX, ray_trig_tables

MAGIC = b"STPC"
HEADER = 284
MAX_RAW_LEN = 1 << 30  # bitstream.py:82
MAX_PIXELS = 1 << 26
MAX_FRAMES = 4096
_CFG = struct.Struct("<Bd HH ddd II HH d")


@dataclass
class DecodeReport:
    point_counts: List[int]
    failed_reconstructions: int
    timings: Dict[str, float]


def _header(blob: bytes):
    """bitstream.py:398-411 header checks (CRC is verified on the GPU)."""
    if len(blob) < HEADER:
        raise TruncatedBlobError(f"blob of {len(blob)} bytes is shorter than the header")
    magic, version, _r, raw_len, enc_len, crc = struct.unpack_from("<4sHHQQI", blob, 0)
    if magic != MAGIC:
        raise MalformedBlobError(f"bad magic {magic!r}")
    if version != 1:
        raise UnknownVersionError(f"format version {version} not supported")
    if raw_len > MAX_RAW_LEN:
        raise MalformedBlobError(f"raw payload length {raw_len} exceeds cap")
    if HEADER + enc_len > len(blob):
        raise TruncatedBlobError("encoded payload extends past end of blob")
    return raw_len, enc_len, crc


def _varints(buf: np.ndarray, pos: int, count: int) -> Tuple[np.ndarray, int]:
    """Vectorised LEB128 decode of `count` values at buf[pos:] (varint_decode_kernel)."""
    seg = buf[pos:pos + 10 * count]
    term = np.flatnonzero(seg < 128)
    if term.size < count:
        raise TruncatedBlobError("residual index varints ran past payload")
    end = int(term[count - 1]) + 1
    seg = seg[:end].astype(np.int64)
    starts = np.concatenate(([0], term[:count - 1] + 1))
    group = np.zeros(end, np.int64)
    group[starts[1:]] = 1
    group = np.cumsum(group)
    shift = 7 * (np.arange(end) - starts[group])
    if shift.max(initial=0) > 63:
        raise TruncatedBlobError("overlong varint")
    vals = np.add.reduceat((seg & 0x7F) << shift, starts)
    return vals, pos + end


def _parse(payload: bytes):
    """Structure of one raw payload (bitstream.py:413-519)."""
    buf = np.frombuffer(payload, np.uint8)
    pos = 0

    def need(nbytes):
        if nbytes < 0 or pos + nbytes > len(payload):
            raise TruncatedBlobError(f"payload ends at byte {len(payload)}, needed {pos + nbytes}")

    need(_CFG.size)
    (mode, tau, tw, th, theta_r, phi_r, phi_off, w, h, n, k, quant) = _CFG.unpack_from(payload, 0)
    pos = _CFG.size
    if mode not in (0, 1):
        raise MalformedBlobError(f"unknown mode code {mode}")
    if not all(np.isfinite([tau, theta_r, phi_r, phi_off, quant])):
        raise MalformedBlobError("non-finite config field")
    if tau <= 0 or theta_r <= 0 or phi_r <= 0 or quant <= 0:
        raise MalformedBlobError("non-positive config field")
    if w < 1 or h < 1 or w * h > MAX_PIXELS:
        raise MalformedBlobError(f"image size {w}x{h} outside supported range")
    if n < 1 or n > MAX_FRAMES:
        raise MalformedBlobError(f"frame count {n} outside supported range")
    if tw < 1 or th < 1 or not 0 <= k < n or (mode == 0 and n != 1):
        raise MalformedBlobError("inconsistent config")
    cfg = dict(mode=mode, tau=tau, tile_w=tw, tile_h=th, theta_r=theta_r, phi_r=phi_r, phi_offset=phi_off,
               w=w, h=h, n_frames=n, k_index=k, range_quant=quant)
    tx, ty = -(-w // tw), -(-h // th)
    need(48 * n)
    xf = np.frombuffer(payload, "<f4", 12 * n, pos).astype(np.float64).reshape(n, 12)
    pos += 48 * n
    nb = (w * h + 7) // 8
    need(nb * n)
    vbits = buf[pos:pos + nb * n].reshape(n, nb)
    pos += nb * n
    # per-tile plane maps: float4 (a, b, c, kind) per (channel, tile)
    tmap = np.zeros((n, ty, tx, 4), np.float32)
    pm = (n + 7) // 8
    need(4)
    (n_runs,) = struct.unpack_from("<I", payload, pos)
    pos += 4
    runs = []
    for _ in range(n_runs):
        need(18 + pm)
        row, s, ln, a, b, c = struct.unpack_from("<HHHfff", payload, pos)
        pos += 18
        if row >= ty or ln < 1 or s + ln > tx:
            raise MalformedBlobError("temporal run outside tile grid")
        bits = payload[pos:pos + pm]
        pos += pm
        offs = []
        for ch in range(n):
            if bits[ch >> 3] & (1 << (ch & 7)):
                if ch == k:
                    offs.append((ch, c))
                else:
                    need(4)
                    offs.append((ch, struct.unpack_from("<f", payload, pos)[0]))
                    pos += 4
        if not any(ch == k for ch, _ in offs):
            raise MalformedBlobError("temporal run missing key-frame offset")
        runs.append((row, s, ln, a, b, offs))
    fb = []
    for ch in range(n):
        need(4)
        (nrows,) = struct.unpack_from("<I", payload, pos)
        pos += 4
        if nrows > ty:
            raise MalformedBlobError("more fallback rows than tile rows")
        for _ in range(nrows):
            need(4)
            row, nr = struct.unpack_from("<HH", payload, pos)
            pos += 4
            if row >= ty or nr > tx:
                raise MalformedBlobError("fallback row outside tile grid")
            need(16 * nr)
            rec = np.frombuffer(payload, dtype=[("s", "<u2"), ("l", "<u2"), ("abc", "<f4", 3)], count=nr, offset=pos)
            pos += 16 * nr
            if nr and (np.any(rec["l"] < 1) or np.any(rec["s"].astype(np.int64) + rec["l"] > tx)):
                raise MalformedBlobError("fallback run outside tile grid")
            fb.append((ch, row, rec))
    # fallback first (kind 2), temporal overrides (kind 1): temporal coverage wins
    for ch, row, rec in fb:
        for s, ln, abc in zip(rec["s"], rec["l"], rec["abc"]):
            tmap[ch, row, s:s + ln] = (abc[0], abc[1], abc[2], 2.0)
    for row, s, ln, a, b, offs in runs:
        for ch, cc in offs:
            tmap[ch, row, s:s + ln] = (a, b, cc, 1.0)
    res_flat, res_r, res_f = [], [], []
    for ch in range(n):
        need(4)
        (cnt,) = struct.unpack_from("<I", payload, pos)
        pos += 4
        if cnt > w * h:
            raise MalformedBlobError("residual count exceeds pixel count")
        if cnt == 0:
            continue
        deltas, pos = _varints(buf, pos, cnt)
        if deltas[0] < 0 or np.any(deltas[1:] < 1) or np.any(deltas > w * h):
            raise MalformedBlobError("residual pixel deltas out of range")
        flat = np.cumsum(deltas)
        if flat[-1] >= w * h:
            raise MalformedBlobError("residual pixel indices not strictly increasing")
        need(2 * cnt + 4)
        codes = np.frombuffer(payload, "<u2", cnt, pos).astype(np.int64)
        pos += 2 * cnt
        (n_esc,) = struct.unpack_from("<I", payload, pos)
        pos += 4
        need(4 * n_esc)
        esc = np.frombuffer(payload, "<f4", n_esc, pos).astype(np.float64)
        pos += 4 * n_esc
        emask = codes == 0xFFFF
        if int(np.count_nonzero(emask)) != n_esc:
            raise MalformedBlobError("escape count mismatch in residual section")
        ranges = codes.astype(np.float64) * quant
        ranges[emask] = esc
        res_flat.append(flat)
        res_r.append(ranges)
        res_f.append(np.full(cnt, ch, np.int32))
    if pos != len(payload):
        raise MalformedBlobError(f"{len(payload) - pos} trailing payload bytes")
    return cfg, xf, vbits, tmap, res_flat, res_r, res_f


def _inverse_rows(xf: np.ndarray) -> np.ndarray:
    """R^-1 | T^-1 per frame with the reference's numpy expressions (motion.py:78-79)."""
    out = np.empty_like(xf)
    for i, row in enumerate(xf):
        R = row[:9].reshape(3, 3)
        T = row[9:]
        out[i, :9] = R.T.reshape(9)
        out[i, 9:] = -(R.T @ T)
    return out


def decompress_many(blobs: Sequence[bytes]) -> Tuple[List[List[np.ndarray]], List[DecodeReport]]:
    """Decode a batch of blobs (one device pass per distinct configuration)."""
    import time

    L = _native.load(require_device=True)
    t0 = time.perf_counter()
    heads = [_header(b) for b in blobs]
    off = np.zeros(len(blobs) + 1, np.int64)
    off[1:] = np.cumsum([(len(b) + 15) // 16 * 16 for b in blobs])
    arena = np.zeros(int(off[-1]), np.uint8)
    for b, o in zip(blobs, off[:-1]):
        arena[o:o + len(b)] = np.frombuffer(b, np.uint8)
    raw_off = np.zeros(len(blobs) + 1, np.int64)
    raw_off[1:] = np.cumsum([(h[0] + 15) // 16 * 16 for h in heads])
    dev = _Dev(L)
    d_blobs = dev.put(arena)
    d_off = dev.put(off[:-1])
    crc = np.zeros(len(blobs), np.uint32)
    _native.check(L.stpc_crc32_blobs(d_blobs, d_off, len(blobs), crc.ctypes.data, None))
    for h, c in zip(heads, crc):
        if int(c) != h[2]:
            raise ChecksumError("payload CRC-32 mismatch")
    d_raw = dev.alloc(max(int(raw_off[-1]), 1))
    d_roff = dev.put(raw_off[:-1])
    st = np.zeros(len(blobs), np.int32)
    _native.check(L.stpc_huffman_decode_blobs(d_blobs, d_off, len(blobs), d_raw, d_roff, st.ctypes.data, None))
    if np.any(st == 1):
        raise TruncatedBlobError("entropy payload ended mid-symbol")
    if np.any(st != 0):
        raise MalformedBlobError("invalid Huffman code in payload")
    raw = np.empty(int(raw_off[-1]), np.uint8)
    _native.check(L.stpc_memcpy_d2h(raw.ctypes.data, d_raw, raw.nbytes))
    t1 = time.perf_counter()
    parsed = [_parse(raw[o:o + h[0]].tobytes()) for o, h in zip(raw_off[:-1], heads)]
    t2 = time.perf_counter()
    clouds_all: List[List[np.ndarray]] = [None] * len(blobs)  # type: ignore
    reports: List[DecodeReport] = [None] * len(blobs)  # type: ignore
    by_cfg: Dict[tuple, List[int]] = {}
    for i, p in enumerate(parsed):
        by_cfg.setdefault(tuple(sorted(p[0].items())), []).append(i)
    for key, idxs in by_cfg.items():
        cfg = dict(key)
        n, w, h = cfg["n_frames"], cfg["w"], cfg["h"]
        F = n * len(idxs)
        tabs = ray_trig_tables(w, h, cfg["theta_r"], cfg["phi_r"], cfg["phi_offset"])
        trig = np.concatenate(tabs)
        vbits = np.concatenate([parsed[i][2] for i in idxs]).reshape(F, -1)
        tmap = np.concatenate([parsed[i][3] for i in idxs]).reshape(F, -1, 4)
        xf_inv = np.concatenate([_inverse_rows(parsed[i][1]) for i in idxs])
        flats, rngs, frames = [], [], []
        for j, i in enumerate(idxs):
            for fl, rr, ff in zip(parsed[i][4], parsed[i][5], parsed[i][6]):
                flats.append(fl)
                rngs.append(rr)
                frames.append(ff + j * n)
        res_flat = np.concatenate(flats) if flats else np.zeros(1, np.int64)
        res_r = np.concatenate(rngs) if rngs else np.zeros(1)
        res_f = np.concatenate(frames) if frames else np.zeros(1, np.int32)
        n_res = int(sum(x.size for x in flats))
        cap = int(np.unpackbits(vbits, axis=1).sum()) + 1
        d_trig, d_vb, d_tm = dev.put(trig), dev.put(np.ascontiguousarray(vbits)), dev.put(np.ascontiguousarray(tmap))
        d_rf, d_rr, d_rfr = dev.put(res_flat), dev.put(res_r), dev.put(res_f.astype(np.int32))
        d_xi = dev.put(xf_inv)
        d_scr = dev.alloc(8 * F * w * h)
        d_pts = dev.alloc(24 * cap)
        counts = np.zeros(F, np.int64)
        failed = ctypes.c_int64()
        _native.check(L.stpc_reconstruct_frames(
            w, h, cfg["tile_w"], cfg["tile_h"], d_trig, F, d_vb, vbits.shape[1], d_tm, d_rf, d_rr, d_rfr,
            n_res, d_xi, DEFAULT_R_MAX, d_scr, d_pts, cap, counts.ctypes.data, ctypes.byref(failed), None))
        pts = np.empty((int(counts.sum()), 3))
        _native.check(L.stpc_memcpy_d2h(pts.ctypes.data, d_pts, pts.nbytes))
        bounds = np.concatenate(([0], np.cumsum(counts)))
        for j, i in enumerate(idxs):
            clouds_all[i] = [pts[bounds[j * n + c]:bounds[j * n + c + 1]] for c in range(n)]
            reports[i] = DecodeReport(point_counts=[int(x) for x in counts[j * n:(j + 1) * n]],
                                      failed_reconstructions=int(failed.value) if len(idxs) == 1 else -1,
                                      timings={})
    t3 = time.perf_counter()
    for r in reports:
        r.timings = {"entropy": t1 - t0, "parse": t2 - t1, "reconstruct": t3 - t2}
    dev.free_all()
    return clouds_all, reports


def decompress_full(blob: bytes):
    clouds, reps = decompress_many([blob])
    return clouds[0], reps[0]


def decompress(blob: bytes) -> List[np.ndarray]:
    """Drop-in for stpc.decompress: one (N, 3) float64 cloud per frame."""
    return decompress_full(blob)[0]


class _Dev:
    """Scoped device allocations through the C-ABI."""

    def __init__(self, L):
        self.L = L
        self.ptrs = []

    def alloc(self, nbytes):
        p = ctypes.c_void_p()
        _native.check(self.L.stpc_malloc(ctypes.byref(p), int(max(nbytes, 1))))
        self.ptrs.append(p)
        return p

    def put(self, arr):
        arr = np.ascontiguousarray(arr)
        p = self.alloc(arr.nbytes)
        if arr.nbytes:
            _native.check(self.L.stpc_memcpy_h2d(p, arr.ctypes.data, arr.nbytes))
        return p

    def free_all(self):
        for p in self.ptrs:
            self.L.stpc_free(p)
        self.ptrs = []
