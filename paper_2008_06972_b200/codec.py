"""Drop-in ``compress`` for the reference's stream/single-frame encoder.

Mirrors the public contract of /root/reference/pkg/src/stpc/bitstream.py:
``CodecConfig`` (:87-126), ``EncodeReport`` (:129-139) and
``compress(clouds, cfg, poses=None, imu_samples=None, frame_times=None,
v0=None, threads=1) -> (bytes, EncodeReport)`` (:527-602), emitting the same
.stpc v1 bytes.  The work runs in libstpc_b200 on the GPU: projection,
spatial and temporal fits, residual compaction, payload assembly, Huffman
coding and CRC.  The host only validates arguments, chains the poses into
float32 transforms (microseconds) and builds the report.

``compress_groups`` is the batch form the reference does not have: many
independent K+P groups per call, the natural unit of throughput.
"""

from __future__ import annotations

import ctypes
import logging
import threading
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .errors import DataError
from .geometry import (
    COND_LIMIT,
    DEFAULT_PHI_OFFSET,
    DEFAULT_R_MAX,
    AngularResolution,
    RigidTransform,
    frame_transforms,
    matmul_contract,
    poses_to_transform_rows,
    poses_to_transforms,
    ray_trig_tables,
)

log = logging.getLogger(__name__)

MODE_SINGLE = "single"
MODE_STREAM = "stream"
_MODE_CODES = {MODE_SINGLE: 0, MODE_STREAM: 1}
HEADER_SIZE = 284


@dataclass(frozen=True)
class TileGrid:
    tile_w: int
    tile_h: int
    width: int
    height: int

    @property
    def tiles_x(self) -> int:
        return -(-self.width // self.tile_w)

    @property
    def tiles_y(self) -> int:
        return -(-self.height // self.tile_h)


@dataclass(frozen=True)
class CodecConfig:
    """Same fields, defaults and validation as the reference CodecConfig."""

    mode: str = MODE_SINGLE
    tau: float = 0.02
    tile_w: int = 4
    tile_h: int = 4
    res: AngularResolution = field(default_factory=AngularResolution)
    phi_offset: float = DEFAULT_PHI_OFFSET
    w: int = 1800
    h: int = 64
    n_frames: int = 1
    k_index: Optional[int] = None
    range_quant: float = 0.005

    def __post_init__(self):
        if self.mode not in _MODE_CODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == MODE_SINGLE and self.n_frames != 1:
            raise ValueError("single-frame mode takes exactly one frame")
        if self.tau <= 0 or self.range_quant <= 0:
            raise ValueError("tau and range_quant must be positive")
        if min(self.tile_w, self.tile_h, self.w, self.h, self.n_frames) < 1:
            raise ValueError("dimensions must be >= 1")
        if self.k_index is None:
            object.__setattr__(self, "k_index", self.n_frames // 2)
        if not (0 <= self.k_index < self.n_frames):
            raise ValueError("k_index out of range")
        if self.range_quant > self.tau / 2:
            log.warning("range_quant %.4g above tau/2 (%.4g); residual error may dominate",
                        self.range_quant, self.tau / 2)

    def grid(self) -> TileGrid:
        return TileGrid(self.tile_w, self.tile_h, self.w, self.h)


@dataclass
class EncodeReport:
    raw_bytes: int
    blob_bytes: int
    compression_rate: float
    point_counts: List[int]
    dropped_points: int
    collision_fractions: List[float]
    coverage: List[Dict[str, int]]
    fractions: Dict[str, float]
    timings: Dict[str, float]
    eps_band_points: int = 0  # binnings within 1e-9 of a bin edge


_new_bytes = ctypes.pythonapi.PyBytes_FromStringAndSize
_new_bytes.restype = ctypes.py_object
_new_bytes.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_bytes_buf = ctypes.pythonapi.PyBytes_AsString
_bytes_buf.restype = ctypes.c_void_p
_bytes_buf.argtypes = [ctypes.py_object]


def _bytes_from_arena(L, base: int, off: np.ndarray, ln: np.ndarray) -> List[bytes]:
    """One bytes object per blob of a host arena.  The objects are allocated
    uninitialised (PyBytes_FromStringAndSize(NULL, n), as CPython's own
    builders do) and filled by one threaded native copy before they are
    returned, so no other code ever sees them unfilled."""
    G = len(ln)
    out = [_new_bytes(None, int(n)) for n in ln]
    if G:
        dst = (ctypes.c_void_p * G)(*[_bytes_buf(b) for b in out])
        src_off = np.ascontiguousarray(off[:G], np.int64)
        lens = np.ascontiguousarray(ln, np.int64)
        _native.check(L.stpc_host_scatter(base, src_off.ctypes.data, lens.ctypes.data, dst, G))
    return out


class Encoder:
    """One native encoder (device workspace + trig tables) per config and
    input dtype; reuse it across calls to amortise allocation."""

    def __init__(self, cfg: CodecConfig, points_f64: bool = False):
        L = _native.load(require_device=True)
        self.cfg = cfg
        self.points_f64 = bool(points_f64)
        c = _native.StpcConfig(
            mode=_MODE_CODES[cfg.mode], tile_w=cfg.tile_w, tile_h=cfg.tile_h, w=cfg.w, h=cfg.h,
            n_frames=cfg.n_frames, k_index=cfg.k_index, points_f64=int(self.points_f64),
            tau=cfg.tau, theta_r=cfg.res.theta_r, phi_r=cfg.res.phi_r, phi_offset=cfg.phi_offset,
            range_quant=cfg.range_quant, r_max=DEFAULT_R_MAX, cond_limit=COND_LIMIT,
        )
        tabs = ray_trig_tables(cfg.w, cfg.h, cfg.res.theta_r, cfg.res.phi_r, cfg.phi_offset)
        self._tabs = tabs
        h = ctypes.c_void_p()
        _native.check(L.stpc_encoder_create(ctypes.byref(c), *[t.ctypes.data for t in tabs], ctypes.byref(h)))
        self._h = h
        self._L = L
        self.lock = threading.Lock()

    def close(self):
        if self._h:
            self._L.stpc_encoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- encode --------------------------------------------------------------
    def encode_device(self, n_groups: int, d_points: int, offsets: np.ndarray,
                      transforms: np.ndarray, stream: int = 0) -> None:
        """Points already in device memory (pointer); blobs stay on device."""
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        xf = np.ascontiguousarray(transforms, dtype=np.float64)
        _native.check(self._L.stpc_encode_device(self._h, n_groups, d_points, off.ctypes.data,
                                                 xf.ctypes.data, stream))

    def encode_host(self, n_groups: int, points: np.ndarray, offsets: np.ndarray,
                    transforms: np.ndarray, out: Optional[np.ndarray] = None, stream: int = 0) -> None:
        """Points in host memory: H2D, encode, and D2H of all blobs into ``out``."""
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        xf = np.ascontiguousarray(transforms, dtype=np.float64)
        out_ptr, cap = (out.ctypes.data, out.nbytes) if out is not None else (None, 0)
        _native.check(self._L.stpc_encode_host(self._h, n_groups, points.ctypes.data, off.ctypes.data,
                                               xf.ctypes.data, out_ptr, cap, stream))

    def encode_host_gather(self, n_groups: int, frames: Sequence[np.ndarray], transforms: np.ndarray,
                           stream: int = 0) -> None:
        """Per-frame host arrays (contiguous (N, 3) of the encoder's dtype):
        gathered natively into pinned staging, pipelined with the encode."""
        n = len(frames)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[a.ctypes.data if a.size else None for a in frames])
        counts = np.array([a.shape[0] if a.size else 0 for a in frames], np.int64)
        xf = np.ascontiguousarray(transforms, dtype=np.float64)
        _native.check(self._L.stpc_encode_host_gather(self._h, n_groups, ptrs, counts.ctypes.data,
                                                      xf.ctypes.data, stream))

    # -- results -------------------------------------------------------------
    def blob_layout(self) -> Tuple[np.ndarray, np.ndarray]:
        G = self._L.stpc_result_groups(self._h)
        off = np.zeros(G + 1, np.int64)
        ln = np.zeros(G, np.int64)
        _native.check(self._L.stpc_result_blobs(self._h, off.ctypes.data, ln.ctypes.data))
        return off, ln

    def blobs(self, arena: Optional[np.ndarray] = None) -> List[bytes]:
        off, ln = self.blob_layout()
        host = self._L.stpc_result_host_blobs(self._h) if arena is None else None
        if host:  # blobs already in the encoder's pinned arena: one parallel copy
            return _bytes_from_arena(self._L, host, off, ln)
        if arena is None:
            arena = np.empty(int(off[-1]), np.uint8)
            _native.check(self._L.stpc_result_copy_blobs(self._h, arena.ctypes.data, arena.nbytes, None))
        return _bytes_from_arena(self._L, arena.ctypes.data, off, ln)

    def frame_stats(self) -> np.ndarray:
        G = self._L.stpc_result_groups(self._h)
        F = G * self.cfg.n_frames
        st = np.zeros((F, _native.STPC_NSTAT), np.int64)
        _native.check(self._L.stpc_result_frame_stats(self._h, st.ctypes.data))
        return st

    def payload_lengths(self) -> np.ndarray:
        G = self._L.stpc_result_groups(self._h)
        out = np.zeros(G, np.int64)
        _native.check(self._L.stpc_result_payload_lengths(self._h, out.ctypes.data))
        return out

    def device_buffer(self, which: int) -> Tuple[int, int]:
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _native.check(self._L.stpc_encoder_buffer(self._h, which, ctypes.byref(p), ctypes.byref(n)))
        return p.value or 0, n.value

    def copy_buffer(self, which: int, dtype, count: int) -> np.ndarray:
        ptr, cap = self.device_buffer(which)
        out = np.empty(count, dtype)
        if out.nbytes > cap:
            raise ValueError("requested more than the buffer holds")
        _native.check(self._L.stpc_memcpy_d2h(out.ctypes.data, ptr, out.nbytes))
        return out


class _Pool:
    """Bounded pool of native contexts (encoders / decoders) keyed by config.

    A call checks a context out (so concurrent calls never share one), and
    returns it afterwards; at most ``max_idle`` idle contexts are kept, least
    recently used evicted first.  Each context holds grow-only device
    workspaces (two F*P fp64 grids for an encoder: ~17 GB at 1024 groups), so
    an unbounded per-thread / per-config cache would exhaust HBM under thread
    pools or config sweeps.  Evicted contexts are dropped, not closed: one
    still referenced elsewhere is freed when its last reference goes."""

    def __init__(self, env: str, default: int):
        import os
        from collections import OrderedDict

        self.max_idle = max(0, int(os.environ.get(env, default)))
        self.idle: "OrderedDict[tuple, List]" = OrderedDict()
        self.lock = threading.Lock()

    def acquire(self, key, factory):
        with self.lock:
            lst = self.idle.get(key)
            if lst:
                obj = lst.pop()
                if not lst:
                    del self.idle[key]
                return obj
        return factory()

    def peek(self, key, factory):
        """The most recently returned idle context of ``key`` (left in the
        pool), created if there is none: how tests read the intermediates of
        the last call."""
        with self.lock:
            lst = self.idle.get(key)
            if lst:
                self.idle.move_to_end(key)
                return lst[-1]
        obj = factory()
        self.release(key, obj)
        return obj

    def release(self, key, obj):
        with self.lock:
            self.idle.setdefault(key, []).append(obj)
            self.idle.move_to_end(key)
            total = sum(len(v) for v in self.idle.values())
            while total > self.max_idle and self.idle:
                k0, lst = next(iter(self.idle.items()))
                lst.pop(0)
                total -= 1
                if not lst:
                    del self.idle[k0]

    def clear(self):
        with self.lock:
            self.idle.clear()


_encoders = _Pool("STPC_ENCODER_POOL", 2)


def get_encoder(cfg: CodecConfig, points_f64: bool = False) -> Encoder:
    """The pooled encoder of ``cfg`` that served the most recent call (or a
    new one)."""
    return _encoders.peek((cfg, bool(points_f64)), lambda: Encoder(cfg, points_f64))


class _checkout:
    def __init__(self, pool: _Pool, key, factory):
        self.pool, self.key, self.factory = pool, key, factory

    def __enter__(self):
        self.obj = self.pool.acquire(self.key, self.factory)
        return self.obj

    def __exit__(self, *exc):
        self.pool.release(self.key, self.obj)
        return False


def release_cached() -> None:
    """Free every idle pooled encoder and decoder (their device workspaces go
    when the last reference does)."""
    from . import decode

    _encoders.clear()
    decode._decoders.clear()


def _transforms_for(cfg: CodecConfig, poses, imu_samples, frame_times, v0) -> List[RigidTransform]:
    """The transform branch of compress (bitstream.py:547-560)."""
    if cfg.n_frames == 1:
        transforms = [RigidTransform.identity()]
    elif poses is not None:
        if len(poses) != cfg.n_frames:
            raise DataError("need one pose per frame")
        transforms = poses_to_transforms(poses, cfg.k_index)
    elif imu_samples is not None:
        if frame_times is None or len(frame_times) != cfg.n_frames:
            raise DataError("IMU alignment needs one frame time per frame")
        transforms = frame_transforms(imu_samples, frame_times, cfg.k_index, v0)
    else:
        raise DataError("stream mode needs poses or IMU samples")
    return [t.round_f32() for t in transforms]


def _stack_points(clouds) -> Tuple[np.ndarray, np.ndarray, bool, List[int]]:
    arrs = [np.asarray(c) for c in clouds]
    counts = []
    f64 = False
    for a in arrs:
        if a.size and (a.ndim != 2 or a.shape[1] != 3):
            raise ValueError("cloud must be an (N, 3) array")
        counts.append(0 if a.size == 0 else a.shape[0])
        if a.size and a.dtype != np.float32:
            f64 = True
    dt = np.float64 if f64 else np.float32
    pts = np.concatenate([a.reshape(-1, 3).astype(dt, copy=False) for a in arrs]) if arrs else np.zeros((0, 3), dt)
    off = np.zeros(len(arrs) + 1, np.int64)
    off[1:] = np.cumsum(counts)
    return np.ascontiguousarray(pts), off, f64, counts


def _frame_arrays(clouds) -> Tuple[List[np.ndarray], bool, List[int]]:
    """Per-frame contiguous (N, 3) arrays of one dtype (float32, or float64
    when any frame is not float32 -- the reference up-casts to float64),
    without concatenating them."""
    arrs = [np.asarray(c) for c in clouds]
    counts = []
    f64 = False
    for a in arrs:
        if a.size and (a.ndim != 2 or a.shape[1] != 3):
            raise ValueError("cloud must be an (N, 3) array")
        counts.append(0 if a.size == 0 else a.shape[0])
        if a.size and a.dtype != np.float32:
            f64 = True
    dt = np.float64 if f64 else np.float32
    frames = [np.ascontiguousarray(a.reshape(-1, 3), dtype=dt) for a in arrs]
    return frames, f64, counts


def _reports(cfg: CodecConfig, stats: np.ndarray, blobs: List[bytes], counts_per_group, timings) -> List[EncodeReport]:
    n = cfg.n_frames
    out = []
    for g, blob in enumerate(blobs):
        st = stats[g * n:(g + 1) * n]
        point_counts = [int(c) for c in counts_per_group[g]]
        raw_bytes = 12 * sum(point_counts)
        kept = st[:, _native.STAT_KEPT]
        valid = st[:, _native.STAT_VALID]
        collisions = kept - valid
        dropped = int((st[:, _native.STAT_REJECTED] + st[:, _native.STAT_DROPPED] + collisions).sum())
        coverage = [
            {"temporal": int(s[_native.STAT_TEMPORAL]), "fallback": int(s[_native.STAT_FALLBACK]),
             "residual": int(s[_native.STAT_RESIDUAL]), "valid": int(s[_native.STAT_VALID])}
            for s in st
        ]
        total_valid = sum(c["valid"] for c in coverage) or 1
        fractions = {
            "temporal": sum(c["temporal"] for c in coverage) / total_valid,
            "spatial": sum(c["fallback"] for c in coverage) / total_valid,
            "residual": sum(c["residual"] for c in coverage) / total_valid,
        }
        coll = [float(c) / float(k) if k > 0 else 0.0 for c, k in zip(collisions, kept)]
        out.append(EncodeReport(
            raw_bytes=raw_bytes, blob_bytes=len(blob),
            compression_rate=raw_bytes / len(blob) if len(blob) else 0.0,
            point_counts=point_counts, dropped_points=dropped, collision_fractions=coll,
            coverage=coverage, fractions=fractions, timings=dict(timings),
            eps_band_points=int(st[:, _native.STAT_EPS_BAND].sum()),
        ))
    return out


def compress_groups(groups: Sequence[Sequence[np.ndarray]], cfg: CodecConfig,
                    poses: Optional[Sequence[Sequence]] = None) -> Tuple[List[bytes], List[EncodeReport]]:
    """Encode many independent groups in one device pass; one blob per group,
    each byte-identical to ``compress(group, cfg, poses=poses[g])``."""
    t0 = time.perf_counter()
    for clouds in groups:
        if len(clouds) != cfg.n_frames:
            raise DataError(f"config expects {cfg.n_frames} frames, got {len(clouds)}")
    if cfg.n_frames > 1 and poses is not None and len(groups):
        if len(poses) != len(groups) or any(len(p) != cfg.n_frames for p in poses):
            raise DataError("need one pose per frame")
        xf = poses_to_transform_rows(poses, cfg.k_index)  # batched, same bits as per group
    else:
        xf = []
        for g, clouds in enumerate(groups):
            ts = _transforms_for(cfg, None if poses is None else poses[g], None, None, None)
            xf.extend(t.row12() for t in ts)
        xf = np.asarray(xf, np.float64).reshape(-1, 12)
    t1 = time.perf_counter()
    frames, f64, counts = _frame_arrays([c for grp in groups for c in grp])
    if f64:
        matmul_contract()  # warns once if this host's BLAS is not the FMA chain
    with _checkout(_encoders, (cfg, f64), lambda: Encoder(cfg, f64)) as enc:
        enc.encode_host_gather(len(groups), frames, xf)
        blobs = enc.blobs()
        stats = enc.frame_stats()
    t2 = time.perf_counter()
    n = cfg.n_frames
    per_group = [counts[g * n:(g + 1) * n] for g in range(len(groups))]
    return blobs, _reports(cfg, stats, blobs, per_group, {"transforms": t1 - t0, "device": t2 - t1})


def compress(clouds: Sequence[np.ndarray], cfg: CodecConfig, poses=None, imu_samples=None,
             frame_times=None, v0=None, threads: int = 1) -> Tuple[bytes, EncodeReport]:
    """Drop-in for stpc.compress: identical blob bytes, GPU execution.
    ``threads`` is accepted for signature compatibility and ignored."""
    if len(clouds) != cfg.n_frames:
        raise DataError(f"config expects {cfg.n_frames} frames, got {len(clouds)}")
    t0 = time.perf_counter()
    if cfg.n_frames > 1 and poses is not None:
        if len(poses) != cfg.n_frames:
            raise DataError("need one pose per frame")
        xf = poses_to_transform_rows([poses], cfg.k_index)  # batched: same bits, no per-frame objects
    else:
        ts = _transforms_for(cfg, poses, imu_samples, frame_times, v0)
        xf = np.asarray([t.row12() for t in ts], np.float64)
    t1 = time.perf_counter()
    pts, off, f64, counts = _stack_points(clouds)
    if f64:
        matmul_contract()  # warns once if this host's BLAS is not the FMA chain
    with _checkout(_encoders, (cfg, f64), lambda: Encoder(cfg, f64)) as enc:
        enc.encode_host(1, pts, off, xf)
        blobs = enc.blobs()
        stats = enc.frame_stats()
    t2 = time.perf_counter()
    rep = _reports(cfg, stats, blobs, [counts], {"transforms": t1 - t0, "device": t2 - t1})
    return blobs[0], rep[0]
