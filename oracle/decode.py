"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the reference decoder.

Restates /root/reference/pkg/src/stpc/bitstream.py ``decompress`` (:605-631):
``deserialize`` (:388-519, CRC :410-411, Huffman huffman.py:80-137), then
``decode_stream_images`` (temporal.py:293-343 with ``reconstruct_span``,
_kernels.py:282-308), ``unproject`` (range_image.py:214-221) and the inverse
frame transform (motion.py:78-79, 70-72).  Used only to check the GPU decoder
(tests/) -- the product never imports it.  Pinned by the hashes of the
reference's own decompress output stored in tests/golden/decoded.npz.
"""

from __future__ import annotations

import ctypes
import struct
import zlib
from dataclasses import dataclass
from typing import List

import numpy as np

from . import oracle as orc

MAX_CODE_LEN = 32


class DecodeFailure(Exception):
    pass


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _lib():
    L = orc.lib()
    if not hasattr(L, "_dec_ready"):
        P, I, Ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.orc_huffman_decode.argtypes = [P, I, I, P, P, P, P, Ci, P]
        L.orc_huffman_decode.restype = Ci
        L.orc_varint_decode.argtypes = [P, I, I, I, P]
        L.orc_varint_decode.restype = I
        L._dec_ready = True
    return L


def huffman_decode(lengths: np.ndarray, encoded: bytes, n: int) -> bytes:
    """huffman.decode_bytes (huffman.py:121-137) with decode_tables (:80-104)."""
    if n == 0:
        return b""
    count = np.zeros(MAX_CODE_LEN + 1, np.int64)
    for s in range(256):
        if lengths[s]:
            count[lengths[s]] += 1
    first = np.zeros(MAX_CODE_LEN + 1, np.int64)
    index = np.zeros(MAX_CODE_LEN + 1, np.int64)
    code = idx = 0
    for ln in range(1, MAX_CODE_LEN + 1):
        first[ln] = code
        index[ln] = idx
        code = (code + count[ln]) << 1
        idx += count[ln]
    symbols = np.array(sorted(np.nonzero(lengths)[0], key=lambda s: (lengths[s], s)), np.uint8)
    enc = np.frombuffer(encoded, np.uint8)
    out = np.empty(n, np.uint8)
    rc = _lib().orc_huffman_decode(_p(np.ascontiguousarray(enc)), enc.size, n, _p(count), _p(first),
                                   _p(index), _p(symbols), MAX_CODE_LEN, _p(out))
    if rc:
        raise DecodeFailure(f"huffman decode failed ({rc})")
    return out.tobytes()


@dataclass
class Decoded:
    cfg: dict
    transforms: list  # (R, T) f64 from the f32 block
    valid: np.ndarray  # (n, h, w) bool
    t_row: list
    t_s: list
    t_len: list
    t_abc: list
    t_off: list  # per run: list of offsets per channel (None = absent)
    fallback: list  # per channel: list of (row, [(s, len, a, b, c)])
    residuals: list  # per channel: (flat idx, ranges)


def deserialize(blob: bytes) -> Decoded:
    magic, version, _r, raw_len, enc_len, crc = struct.unpack_from("<4sHHQQI", blob, 0)
    if magic != b"STPC" or version != 1:
        raise DecodeFailure("bad header")
    lengths = np.frombuffer(blob, np.uint8, 256, 28)
    encoded = blob[284:284 + enc_len]
    if zlib.crc32(encoded) & 0xFFFFFFFF != crc:
        raise DecodeFailure("crc")
    payload = huffman_decode(lengths, encoded, raw_len)
    pos = 0

    def take(fmt):
        nonlocal pos
        vals = struct.unpack_from(fmt, payload, pos)
        pos += struct.calcsize(fmt)
        return vals

    (mode, tau, tw, th, theta_r, phi_r, phi_off, w, h, n, k, quant) = take("<Bd HH ddd II HH d")
    cfg = dict(mode=mode, tau=tau, tile_w=tw, tile_h=th, theta_r=theta_r, phi_r=phi_r,
               phi_offset=phi_off, w=w, h=h, n_frames=n, k_index=k, range_quant=quant)
    tx, ty = -(-w // tw), -(-h // th)
    block = np.frombuffer(payload, "<f4", 12 * n, pos).astype(np.float64).reshape(n, 12)
    pos += 48 * n
    transforms = [(block[i, :9].reshape(3, 3), block[i, 9:]) for i in range(n)]
    nb = (w * h + 7) // 8
    valid = np.empty((n, h, w), bool)
    for ch in range(n):
        valid[ch] = np.unpackbits(np.frombuffer(payload, np.uint8, nb, pos))[: w * h].reshape(h, w).astype(bool)
        pos += nb
    pm = (n + 7) // 8
    (n_runs,) = take("<I")
    t_row, t_s, t_len, t_abc, t_off = [], [], [], [], []
    for _ in range(n_runs):
        row, s, ln, a, b, c = take("<HHHfff")
        bits = payload[pos:pos + pm]
        pos += pm
        offs = [None] * n
        for ch in range(n):
            if bits[ch >> 3] & (1 << (ch & 7)):
                if ch == k:
                    offs[ch] = float(c)
                else:
                    offs[ch] = float(take("<f")[0])
        t_row.append(row), t_s.append(s), t_len.append(ln), t_abc.append((float(a), float(b), float(c)))
        t_off.append(offs)
    fallback = []
    for ch in range(n):
        (nrows,) = take("<I")
        rows = []
        for _ in range(nrows):
            row, nr = take("<HH")
            rows.append((row, [take("<HHfff") for _ in range(nr)]))
        fallback.append(rows)
    residuals = []
    buf = np.frombuffer(payload, np.uint8)
    for ch in range(n):
        (cnt,) = take("<I")
        if cnt == 0:
            residuals.append((np.zeros(0, np.int64), np.zeros(0)))
            continue
        deltas = np.empty(cnt, np.int64)
        end = _lib().orc_varint_decode(_p(buf), buf.size, pos, cnt, _p(deltas))
        if end < 0:
            raise DecodeFailure("varint")
        pos = end
        flat = np.cumsum(deltas)
        codes = np.frombuffer(payload, "<u2", cnt, pos).astype(np.int64)
        pos += 2 * cnt
        (n_esc,) = take("<I")
        esc = np.frombuffer(payload, "<f4", n_esc, pos).astype(np.float64)
        pos += 4 * n_esc
        ranges = codes.astype(np.float64) * quant
        ranges[codes == 0xFFFF] = esc
        residuals.append((flat, ranges))
    if pos != len(payload):
        raise DecodeFailure("trailing bytes")
    return Decoded(cfg, transforms, valid, t_row, t_s, t_len, t_abc, t_off, fallback, residuals)


def reconstruct(rng_out, msk_out, allowed, dirs, v0, u0, u1, a, b, c, r_max=200.0):
    """reconstruct_span (_kernels.py:282-308), vectorised; returns failures."""
    d = dirs[v0:v0 + allowed.shape[0], u0:u1]
    den = (d[..., 0] + a * d[..., 1]) + b * d[..., 2]
    with np.errstate(all="ignore"):
        r_hat = c / den
    good = allowed & (np.abs(den) >= 1e-12) & ~(r_hat <= 0.0) & ~(r_hat > r_max)
    fail = int(np.count_nonzero(allowed & ~good))
    sub_r = rng_out[v0:v0 + allowed.shape[0], u0:u1]
    sub_m = msk_out[v0:v0 + allowed.shape[0], u0:u1]
    sub_r[good] = r_hat[good]
    sub_m[good] = True
    return fail


def decompress(blob: bytes) -> List[np.ndarray]:
    return decompress_full(blob)[0]


def decompress_full(blob: bytes):
    """(clouds, failed reconstructions) as stpc.decompress_full
    (bitstream.py:605-625): runs are applied in stream order, the last
    successful reconstruction of a pixel wins, and every failed (run, pixel)
    counts (temporal.py:307-331)."""
    dec = deserialize(blob)
    failed = 0
    c = dec.cfg
    n, w, h, tw, th = c["n_frames"], c["w"], c["h"], c["tile_w"], c["tile_h"]
    tx, ty = -(-w // tw), -(-h // th)
    dirs = orc.ray_grid(w, h, c["theta_r"], c["phi_r"], c["phi_offset"])
    out = []
    for ch in range(n):
        valid = dec.valid[ch]
        rng_out = np.zeros((h, w))
        msk_out = np.zeros((h, w), bool)
        cov = np.zeros((ty, tx), bool)
        for j, offs in enumerate(dec.t_off):
            if offs[ch] is not None:
                cov[dec.t_row[j], dec.t_s[j]:dec.t_s[j] + dec.t_len[j]] = True
        t_cov = np.repeat(np.repeat(cov, th, 0)[:h], tw, 1)[:, :w]
        for j, offs in enumerate(dec.t_off):
            if offs[ch] is None:
                continue
            v0 = dec.t_row[j] * th
            v1 = min(v0 + th, h)
            u0 = dec.t_s[j] * tw
            u1 = min((dec.t_s[j] + dec.t_len[j]) * tw, w)
            a, b, _ = dec.t_abc[j]
            failed += reconstruct(rng_out, msk_out, valid[v0:v1, u0:u1].copy(), dirs, v0, u0, u1, a, b, offs[ch])
        remaining = valid & ~t_cov
        for row, runs in dec.fallback[ch]:
            v0 = row * th
            v1 = min(v0 + th, h)
            for s, ln, a, b, cc in runs:
                u0 = s * tw
                u1 = min((s + ln) * tw, w)
                failed += reconstruct(rng_out, msk_out, remaining[v0:v1, u0:u1].copy(), dirs, v0, u0, u1,
                                      float(a), float(b), float(cc))
        flat, ranges = dec.residuals[ch]
        if flat.size:
            rng_out.reshape(-1)[flat] = ranges
            msk_out.reshape(-1)[flat] = True
        pts = rng_out[msk_out, None] * dirs[msk_out]
        R, T = dec.transforms[ch]
        Rinv = R.T
        Tinv = -(R.T @ T)
        out.append(orc.transform(pts, Rinv, Tinv))  # pts @ Rinv.T + Tinv (motion.py:70-72)
    return out, failed
