"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the stpc compression hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module; the product package never
does.  It restates the reference's ``compress`` pipeline
(/root/reference/pkg/src/stpc/bitstream.py:527-602) on top of the plain-C
kernel restatement in oracle/stpc_oracle.c:

    transforms  poses_to_transforms + round_f32   motion.py:214-226, 87-92
    convert     RigidTransform.apply + project      motion.py:70-72, range_image.py:165-211
    pass 1      encode_tile_row on the key channel  temporal.py:127-154
    refit       refit_spans per P-channel           temporal.py:142-151
    pass 2      encode_tile_row on ``remaining``    temporal.py:174-201
    residuals   residual_pixels_for_tiles           temporal.py:206-245, spatial.py:160-168
    serialize   .stpc v1 payload + Huffman + CRC    bitstream.py:193-289, huffman.py:23-118

Parity pin: oracle/validate_reference.py compares this oracle byte-for-byte
with the live reference package on BASELINE-shaped inputs, and
tests/test_oracle_golden.py checks it against fixtures the reference itself
produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import heapq
import os
import struct
import subprocess
import zlib
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libstpc_oracle.so")

COND_LIMIT = 1e8  # plane.py:26
R_MAX = 200.0  # range_image.py:34
ESCAPE_U16 = 0xFFFF  # bitstream.py:79
MAX_CODE_LEN = 32  # huffman.py:20


def build(force: bool = False) -> str:
    """Compile the C restatement (no FMA contraction; same libm as numba)."""
    src = os.path.join(HERE, "stpc_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
             "-o", LIB_PATH, src, "-lm"]
        )
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        L.orc_transform.argtypes = [P, I, P, P, P]
        L.orc_project.argtypes = [P, I, D, D, D, I, I, P, P, P]
        L.orc_plane_from_sums.argtypes = [P, D, P]
        L.orc_plane_from_sums.restype = ctypes.c_int
        L.orc_encode_tile_row.argtypes = [P, P, P, I, I, I, I, D, D, D, P, P, P, P]
        L.orc_encode_tile_row.restype = I
        L.orc_refit_spans.argtypes = [P, P, P, I, I, I, I, P, P, P, I, D, D, P, P]
        L.orc_varint_encode.argtypes = [P, I, P]
        L.orc_varint_encode.restype = I
        L.orc_huffman_pack.argtypes = [P, I, P, P, P]
        L.orc_huffman_pack.restype = I
        L.orc_histogram.argtypes = [P, I, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class OracleConfig:
    """The reference CodecConfig fields (bitstream.py:87-126)."""

    mode: str
    tau: float
    tile_w: int
    tile_h: int
    theta_r: float
    phi_r: float
    phi_offset: float
    w: int
    h: int
    n_frames: int
    k_index: int
    range_quant: float = 0.005

    @classmethod
    def of(cls, cfg) -> "OracleConfig":
        res = getattr(cfg, "res", None)
        return cls(
            mode=cfg.mode, tau=float(cfg.tau), tile_w=int(cfg.tile_w), tile_h=int(cfg.tile_h),
            theta_r=float(res.theta_r if res is not None else cfg.theta_r),
            phi_r=float(res.phi_r if res is not None else cfg.phi_r),
            phi_offset=float(cfg.phi_offset), w=int(cfg.w), h=int(cfg.h),
            n_frames=int(cfg.n_frames), k_index=int(cfg.k_index),
            range_quant=float(cfg.range_quant),
        )

    @property
    def tiles_x(self):
        return -(-self.w // self.tile_w)

    @property
    def tiles_y(self):
        return -(-self.h // self.tile_h)


# --------------------------------------------------------------------------
# host geometry (motion.py / range_image.py restatements)
# --------------------------------------------------------------------------


def ray_grid(w, h, theta_r, phi_r, phi_offset) -> np.ndarray:
    """pixel_ray_grid (range_image.py:132-152): same numpy expressions, so the
    same bits on the same host."""
    theta = (np.arange(w, dtype=np.float64) + 0.5) * theta_r
    phi = phi_offset + (np.arange(h, dtype=np.float64) + 0.5) * phi_r
    sin_phi = np.sin(phi)[:, None]
    g = np.empty((h, w, 3), dtype=np.float64)
    g[:, :, 0] = sin_phi * np.sin(theta)[None, :]
    g[:, :, 1] = sin_phi * np.cos(theta)[None, :]
    g[:, :, 2] = np.cos(phi)[:, None]
    return g


def poses_to_transforms(poses, k):
    """G_k^-1 . G_i per frame (motion.py:214-226, compose :74-76, inverse
    :78-79), then round_f32 (:87-92).  poses are (R, T) frame->world."""
    Rk, Tk = (np.asarray(poses[k][0], np.float64), np.asarray(poses[k][1], np.float64).reshape(3))
    Rinv = Rk.T
    Tinv = -(Rk.T @ Tk)
    out = []
    for i, (R, T) in enumerate(poses):
        if i == k:
            Ro, To = np.eye(3), np.zeros(3)
        else:
            R = np.asarray(R, np.float64)
            T = np.asarray(T, np.float64).reshape(3)
            Ro, To = Rinv @ R, Rinv @ T + Tinv
        out.append((Ro.astype(np.float32).astype(np.float64), To.astype(np.float32).astype(np.float64)))
    return out


def transform(pts: np.ndarray, R, T) -> np.ndarray:
    """RigidTransform.apply (motion.py:70-72) via orc_transform's FMA chain."""
    p = np.ascontiguousarray(np.asarray(pts, np.float64).reshape(-1, 3))
    out = np.empty_like(p)
    lib().orc_transform(_p(p), p.shape[0], _p(np.ascontiguousarray(R, np.float64)),
                        _p(np.ascontiguousarray(T, np.float64)), _p(out))
    return out


def convert(cloud: np.ndarray, R, T, cfg: OracleConfig):
    """Transform + project (motion.py:70-72 -> range_image.py:165-211)."""
    pts = np.ascontiguousarray(np.asarray(cloud).reshape(-1, 3))
    n = pts.shape[0]
    p64 = transform(pts, R, T)
    best = np.full(cfg.h * cfg.w, np.inf)
    win = np.full(cfg.h * cfg.w, -1, np.int64)
    counts = np.zeros(3, np.int64)
    lib().orc_project(_p(p64), n, cfg.theta_r, cfg.phi_r, cfg.phi_offset, cfg.w, cfg.h,
                      _p(best), _p(win), _p(counts))
    return best, win, counts


def encode_tile_row(rng, msk, dirs, cfg, tr, tau):
    v0 = tr * cfg.tile_h
    v1 = min(v0 + cfg.tile_h, cfg.h)
    tx = cfg.tiles_x
    run_s = np.zeros(tx, np.int32)
    run_len = np.zeros(tx, np.int32)
    run_abc = np.zeros((tx, 3))
    resid = np.zeros(tx, np.uint8)
    n = lib().orc_encode_tile_row(_p(rng), _p(msk), _p(dirs), cfg.w, v0, v1, cfg.tile_w,
                                  tau, R_MAX, COND_LIMIT, _p(run_s), _p(run_len), _p(run_abc), _p(resid))
    return run_s[:n].copy(), run_len[:n].copy(), run_abc[:n].copy(), resid.astype(bool)


def refit_spans(rng, msk, dirs, cfg, tr, s, ln, abc, tau):
    v0 = tr * cfg.tile_h
    v1 = min(v0 + cfg.tile_h, cfg.h)
    n = s.shape[0]
    ok = np.zeros(n, np.uint8)
    c = np.zeros(n)
    lib().orc_refit_spans(_p(rng), _p(msk), _p(dirs), cfg.w, v0, v1, cfg.tile_w,
                          _p(np.ascontiguousarray(s)), _p(np.ascontiguousarray(ln)),
                          _p(np.ascontiguousarray(abc)), n, tau, R_MAX, _p(ok), _p(c))
    return ok.astype(bool), c


# --------------------------------------------------------------------------
# encode_stream restatement (temporal.py:105-266) on flat arrays
# --------------------------------------------------------------------------


@dataclass
class OracleEncoding:
    """Flat form of the reference's StreamEncoded."""

    k: int
    valid: np.ndarray  # (n, h, w) bool
    ranges: np.ndarray  # (n, h, w) f64, 0 where invalid
    best: np.ndarray  # (n, h*w) f64, inf where empty (project_kernel's grid)
    win: np.ndarray  # (n, h*w) int64
    counts: np.ndarray  # (n, 3) rejected, dropped, kept
    transforms: list  # (R, T) per frame, f32-exact
    # temporal runs, tile-row then s order: row, s, len, abc (n_runs,3), offsets (n_runs, n) nan=None
    t_row: np.ndarray
    t_s: np.ndarray
    t_len: np.ndarray
    t_abc: np.ndarray
    t_off: np.ndarray
    k_resid: List[np.ndarray]  # per tile-row bool[tiles_x]
    # fallback: per channel list of (row, s[], len[], abc[]) for non-empty rows
    fallback: List[list]
    p2_resid: dict  # (ch, tr) -> bool[tiles_x]
    residual_flat: List[np.ndarray]  # per channel sorted flat indices
    residual_r: List[np.ndarray]


def encode_stream(clouds, transforms, cfg: OracleConfig) -> OracleEncoding:
    n, k = cfg.n_frames, cfg.k_index
    tau = cfg.tau
    dirs = ray_grid(cfg.w, cfg.h, cfg.theta_r, cfg.phi_r, cfg.phi_offset)
    best, win, counts = [], [], []
    for i, cloud in enumerate(clouds):
        b, wn, c = convert(cloud, *transforms[i], cfg)
        best.append(b)
        win.append(wn)
        counts.append(c)
    best = np.stack(best)
    valid = np.isfinite(best).reshape(n, cfg.h, cfg.w)
    ranges = np.where(valid.reshape(n, -1), best, 0.0).reshape(n, cfg.h, cfg.w)
    msk = [np.ascontiguousarray(valid[i]).view(np.uint8) for i in range(n)]
    rng = [np.ascontiguousarray(ranges[i]) for i in range(n)]

    t_row, t_s, t_len, t_abc, t_off, k_resid = [], [], [], [], [], []
    for tr in range(cfg.tiles_y):
        s, ln, abc, resid = encode_tile_row(rng[k], msk[k], dirs, cfg, tr, tau)
        k_resid.append(resid)
        off = np.full((s.shape[0], n), np.nan)
        if s.shape[0]:
            off[:, k] = abc[:, 2]
            for ch in range(n):
                if ch == k:
                    continue
                ok, c = refit_spans(rng[ch], msk[ch], dirs, cfg, tr, s, ln, abc, tau)
                off[ok, ch] = c[ok]
        t_row.append(np.full(s.shape[0], tr, np.int64))
        t_s.append(s)
        t_len.append(ln)
        t_abc.append(abc)
        t_off.append(off)
    t_row = np.concatenate(t_row)
    t_s = np.concatenate(t_s).astype(np.int64)
    t_len = np.concatenate(t_len).astype(np.int64)
    t_abc = np.concatenate(t_abc).reshape(-1, 3)
    t_off = np.concatenate(t_off).reshape(-1, n)

    def tile_cover(ch):
        cov = np.zeros((cfg.tiles_y, cfg.tiles_x), bool)
        for j in np.nonzero(~np.isnan(t_off[:, ch]))[0]:
            cov[t_row[j], t_s[j]:t_s[j] + t_len[j]] = True
        return cov

    def expand(tmask):
        return np.repeat(np.repeat(tmask, cfg.tile_h, 0)[:cfg.h], cfg.tile_w, 1)[:, :cfg.w]

    fallback = [[] for _ in range(n)]
    p2_resid = {}
    res_flat: List[np.ndarray] = [np.zeros(0, np.int64)] * n
    res_r: List[np.ndarray] = [np.zeros(0)] * n

    def residual_of(mask2d, resid_rows):
        """Valid pixels of flagged tiles, row-major (spatial.py:160-168)."""
        tm = np.stack(resid_rows) if resid_rows else np.zeros((cfg.tiles_y, cfg.tiles_x), bool)
        sel = mask2d & expand(tm)
        flat = np.flatnonzero(sel.reshape(-1))
        return flat

    res_flat[k] = residual_of(valid[k], k_resid)
    res_r[k] = ranges[k].reshape(-1)[res_flat[k]]
    for ch in range(n):
        if ch == k:
            continue
        remaining = valid[ch] & ~expand(tile_cover(ch))
        rm = np.ascontiguousarray(remaining).view(np.uint8)
        rows = []
        for tr in range(cfg.tiles_y):
            s, ln, abc, resid = encode_tile_row(rng[ch], rm, dirs, cfg, tr, tau)
            p2_resid[(ch, tr)] = resid
            rows.append(resid)
            if s.shape[0]:
                fallback[ch].append((tr, s, ln, abc))
        res_flat[ch] = residual_of(remaining, rows)
        res_r[ch] = ranges[ch].reshape(-1)[res_flat[ch]]

    return OracleEncoding(
        k=k, valid=valid, ranges=ranges, best=best, win=np.stack(win), counts=np.stack(counts),
        transforms=transforms, t_row=t_row, t_s=t_s, t_len=t_len, t_abc=t_abc, t_off=t_off,
        k_resid=k_resid, fallback=fallback, p2_resid=p2_resid,
        residual_flat=res_flat, residual_r=res_r,
    )


# --------------------------------------------------------------------------
# .stpc v1 serialization (bitstream.py:193-289, README.md:79-120)
# --------------------------------------------------------------------------

_CONFIG_FMT = "<Bd HH ddd II HH d"  # bitstream.py:142-157


def config_bytes(cfg: OracleConfig) -> bytes:
    return struct.pack(
        _CONFIG_FMT, 0 if cfg.mode == "single" else 1, cfg.tau, cfg.tile_w, cfg.tile_h,
        cfg.theta_r, cfg.phi_r, cfg.phi_offset, cfg.w, cfg.h, cfg.n_frames, cfg.k_index,
        cfg.range_quant,
    )


def varint_bytes(vals: np.ndarray) -> bytes:
    if vals.size == 0:
        return b""
    out = np.empty(vals.size * 10, np.uint8)
    v = np.ascontiguousarray(vals.astype(np.int64))
    m = lib().orc_varint_encode(_p(v), v.size, _p(out))
    return out[:m].tobytes()


def payload_bytes(enc: OracleEncoding, cfg: OracleConfig) -> bytes:
    n, k = cfg.n_frames, enc.k
    out = bytearray(config_bytes(cfg))
    tr_block = np.empty((n, 12), "<f4")
    for i, (R, T) in enumerate(enc.transforms):
        tr_block[i, :9] = np.asarray(R).reshape(9)
        tr_block[i, 9:] = np.asarray(T)
    out += tr_block.tobytes()
    for ch in range(n):
        out += np.packbits(enc.valid[ch].reshape(-1)).tobytes()

    # temporal runs: <HHH fff> + LSB-first presence bits + f32 per present P channel
    pm = (n + 7) // 8
    out += struct.pack("<I", enc.t_s.shape[0])
    present = ~np.isnan(enc.t_off)
    for j in range(enc.t_s.shape[0]):
        a, b, c = (np.float32(x) for x in enc.t_abc[j])
        out += struct.pack("<HHHfff", enc.t_row[j], enc.t_s[j], enc.t_len[j], a, b, c)
        bits = np.zeros(pm, np.uint8)
        chs = np.nonzero(present[j])[0]
        for ch in chs:
            bits[ch >> 3] |= np.uint8(1 << (ch & 7))
        out += bits.tobytes()
        extra = [enc.t_off[j, ch] for ch in chs if ch != k]
        out += np.asarray(extra, "<f4").tobytes()

    for ch in range(n):
        rows = enc.fallback[ch]
        out += struct.pack("<I", len(rows))
        for tr, s, ln, abc in rows:
            out += struct.pack("<HH", tr, s.shape[0])
            rec = np.zeros(s.shape[0], dtype=[("s", "<u2"), ("l", "<u2"), ("abc", "<f4", 3)])
            rec["s"] = s
            rec["l"] = ln
            rec["abc"] = abc
            out += rec.tobytes()

    for ch in range(n):
        flat = enc.residual_flat[ch]
        out += struct.pack("<I", flat.size)
        if flat.size:
            deltas = np.diff(flat, prepend=0)
            out += varint_bytes(deltas)
            q = np.rint(enc.residual_r[ch] / cfg.range_quant).astype(np.int64)
            esc = (q < 1) | (q >= ESCAPE_U16)
            out += np.where(esc, ESCAPE_U16, q).astype("<u2").tobytes()
            out += struct.pack("<I", int(esc.sum()))
            out += enc.residual_r[ch][esc].astype("<f4").tobytes()
    return bytes(out)


def code_lengths(freqs: np.ndarray) -> np.ndarray:
    """huffman.code_lengths_from_counts (huffman.py:23-60): heap merges ordered
    by (weight, serial) with leaf serial = symbol, internal serials 256, 257...;
    lengths capped at 32 with the Kraft repair."""
    lengths = np.zeros(256, np.uint8)
    syms = [int(s) for s in np.nonzero(freqs)[0]]
    if not syms:
        return lengths
    if len(syms) == 1:
        lengths[syms[0]] = 1
        return lengths
    heap = [(int(freqs[s]), s, (s,)) for s in syms]
    heapq.heapify(heap)
    depth = dict.fromkeys(syms, 0)
    serial = 256
    while len(heap) > 1:
        w1, _, m1 = heapq.heappop(heap)
        w2, _, m2 = heapq.heappop(heap)
        for s in m1 + m2:
            depth[s] += 1
        heapq.heappush(heap, (w1 + w2, serial, m1 + m2))
        serial += 1
    for s, d in depth.items():
        lengths[s] = d
    if lengths.max() > MAX_CODE_LEN:
        L = np.minimum(lengths.astype(np.int64), MAX_CODE_LEN)
        # kraft in units of 2^-32 is exact (the reference's float sum is exact too)
        kraft = int(sum(1 << (MAX_CODE_LEN - int(l)) for l in L if l > 0))
        while kraft > (1 << MAX_CODE_LEN):
            cand = np.nonzero((L > 0) & (L < MAX_CODE_LEN))[0]
            pick = cand[np.argmax(L[cand])]
            kraft -= 1 << (MAX_CODE_LEN - int(L[pick]))
            L[pick] += 1
            kraft += 1 << (MAX_CODE_LEN - int(L[pick]))
        lengths = L.astype(np.uint8)
    return lengths


def canonical_codes(lengths: np.ndarray) -> np.ndarray:
    """huffman.canonical_codes (huffman.py:63-77)."""
    codes = np.zeros(256, np.int64)
    code, prev = 0, 0
    for s in sorted(np.nonzero(lengths)[0], key=lambda s: (lengths[s], s)):
        ln = int(lengths[s])
        code <<= ln - prev
        codes[s] = code
        code += 1
        prev = ln
    return codes


def histogram(payload: bytes) -> np.ndarray:
    data = np.frombuffer(payload, np.uint8)
    h = np.zeros(256, np.int64)
    lib().orc_histogram(_p(np.ascontiguousarray(data)), data.size, _p(h))
    return h


def entropy_blob(payload: bytes) -> bytes:
    """huffman.encode_bytes + header (huffman.py:107-118; bitstream.py:279-289)."""
    data = np.frombuffer(payload, np.uint8)
    if data.size:
        freqs = histogram(payload)
        lengths = code_lengths(freqs)
        codes = canonical_codes(lengths)
        out = np.empty((int(lengths.max()) * data.size + 7) // 8 + 8, np.uint8)
        m = lib().orc_huffman_pack(_p(np.ascontiguousarray(data)), data.size, _p(codes),
                                   _p(lengths.astype(np.int64)), _p(out))
        encoded = out[:m].tobytes()
    else:
        lengths = np.zeros(256, np.uint8)
        encoded = b""
    header = struct.pack("<4sHHQQI", b"STPC", 1, 0, len(payload), len(encoded),
                         zlib.crc32(encoded) & 0xFFFFFFFF)
    return header + lengths.tobytes() + encoded


def compress(clouds: Sequence[np.ndarray], cfg, poses=None):
    """Oracle of the reference ``compress`` for the poses path (or n == 1).

    Returns (blob, OracleEncoding)."""
    ocfg = cfg if isinstance(cfg, OracleConfig) else OracleConfig.of(cfg)
    if len(clouds) != ocfg.n_frames:
        raise ValueError("frame count mismatch")
    if ocfg.n_frames == 1:
        transforms = [(np.eye(3), np.zeros(3))]
    else:
        transforms = poses_to_transforms(poses, ocfg.k_index)
    enc = encode_stream(clouds, transforms, ocfg)
    return entropy_blob(payload_bytes(enc, ocfg)), enc
