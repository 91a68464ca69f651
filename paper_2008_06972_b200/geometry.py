"""Host-side geometry of the drop-in API (microsecond-scale, numpy).

Everything here runs once per frame or per group on a handful of numbers and
feeds the device path: the angular resolution type, rigid transforms and
their frame->key-frame chaining, IMU dead reckoning, and the trig tables of
the pixel-centre ray grid.  The expressions are evaluated with the same numpy
operations, in the same order, as the reference
(/root/reference/pkg/src/stpc/motion.py, range_image.py), so the float32
transforms written into the blob are bit-identical.
"""

from __future__ import annotations

import bisect
import logging
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .errors import DataError, ImuCoverageError

log = logging.getLogger(__name__)

DEFAULT_THETA_R = 2.0 * np.pi / 1800.0  # range_image.py:29
DEFAULT_PHI_R = 0.00698  # range_image.py:30
DEFAULT_PHI_OFFSET = 1.48  # range_image.py:31
DEFAULT_R_MAX = 200.0  # range_image.py:34
COND_LIMIT = 1e8  # plane.py:26
ORTHONORMAL_ATOL = 1e-6  # motion.py:37


@dataclass(frozen=True)
class AngularResolution:
    """Horizontal / vertical angular step per pixel (range_image.py:37-46)."""

    theta_r: float = DEFAULT_THETA_R
    phi_r: float = DEFAULT_PHI_R

    def __post_init__(self):
        if not (self.theta_r > 0.0 and self.phi_r > 0.0):
            raise ValueError("angular resolutions must be positive")


@dataclass(frozen=True)
class ImuSample:
    t: float
    accel: np.ndarray
    gyro: np.ndarray


class RigidTransform:
    """p' = R p + T (motion.py:49-99 semantics: compose, inverse, round_f32)."""

    __slots__ = ("R", "T")

    def __init__(self, R, T):
        R = np.asarray(R, dtype=np.float64)
        T = np.asarray(T, dtype=np.float64).reshape(3)
        if R.shape != (3, 3):
            raise ValueError("R must be 3x3")
        if not np.allclose(R.T @ R, np.eye(3), atol=ORTHONORMAL_ATOL):
            raise ValueError("R is not orthonormal")
        if not np.isclose(np.linalg.det(R), 1.0, atol=ORTHONORMAL_ATOL):
            raise ValueError("R must be a proper rotation (det +1)")
        self.R = R
        self.T = T

    @classmethod
    def identity(cls) -> "RigidTransform":
        return cls(np.eye(3), np.zeros(3))

    @classmethod
    def of(cls, pose) -> "RigidTransform":
        """Accept a RigidTransform-like object (``.R``/``.T``) or an (R, T) pair."""
        if isinstance(pose, RigidTransform):
            return pose
        if hasattr(pose, "R") and hasattr(pose, "T"):
            return cls(pose.R, pose.T)
        R, T = pose
        return cls(R, T)

    def compose(self, other: "RigidTransform") -> "RigidTransform":
        return RigidTransform(self.R @ other.R, self.R @ other.T + self.T)

    def inverse(self) -> "RigidTransform":
        return RigidTransform(self.R.T, -(self.R.T @ self.T))

    def round_f32(self) -> "RigidTransform":
        return RigidTransform(self.R.astype(np.float32).astype(np.float64),
                              self.T.astype(np.float32).astype(np.float64))

    def apply(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.R.T + self.T

    def row12(self) -> np.ndarray:
        return np.concatenate([self.R.reshape(9), self.T])

    def __eq__(self, other):
        return isinstance(other, RigidTransform) and np.array_equal(self.R, other.R) and np.array_equal(self.T, other.T)


_MATMUL_CONTRACT: Optional[str] = None


def matmul_contract() -> str:
    """How this host's numpy evaluates RigidTransform.apply (pts @ R.T + T,
    motion.py:70-72) per output coordinate: "fma" when it equals
    fma(z, r2, fma(y, r1, x*r0)) -- the BLAS dgemm micro-kernel's FMA chain,
    which the device reproduces (common.cuh xform_coord) -- "plain" when it
    equals ((x*r0 + y*r1) + z*r2), "mixed" otherwise.  Only float64 clouds that
    are not float32-representable can tell them apart (float32 products are
    exact); the reference's own bits for those then depend on the host's BLAS,
    and the device matches them where this returns "fma".  Probed once on
    2000 points with exact rational arithmetic for the FMA reference."""
    global _MATMUL_CONTRACT
    if _MATMUL_CONTRACT is None:
        from fractions import Fraction

        rng = np.random.default_rng(12345)
        p = rng.uniform(-60.0, 60.0, (2000, 3)) * (1.0 + rng.uniform(-1e-6, 1e-6, (2000, 3)))
        R = rng.uniform(-1.0, 1.0, (3, 3)).astype(np.float32).astype(np.float64)
        out = p @ R.T
        fma = plain = True
        for i in range(p.shape[0]):
            x, y, z = (float(v) for v in p[i])
            for j in range(3):
                r0, r1, r2 = (float(v) for v in R[j])
                inner = float(Fraction(y) * Fraction(r1) + Fraction(x * r0))
                f = float(Fraction(z) * Fraction(r2) + Fraction(inner))
                fma &= bool(out[i, j] == f)
                plain &= bool(out[i, j] == (x * r0 + y * r1) + z * r2)
        _MATMUL_CONTRACT = "fma" if fma else ("plain" if plain else "mixed")
        if _MATMUL_CONTRACT != "fma":
            log.warning("numpy matmul on this host is %r, not the FMA chain the device reproduces: blobs of "
                        "float64 clouds that are not float32-representable may differ in the last bits from a "
                        "reference run on this host (float32 clouds are unaffected)", _MATMUL_CONTRACT)
    return _MATMUL_CONTRACT


def poses_to_transforms(poses: Sequence, k_index: int) -> List[RigidTransform]:
    """Frame -> key-frame transforms G_k^-1 . G_i from frame -> world poses
    (motion.py:214-226)."""
    poses = [RigidTransform.of(p) for p in poses]
    inv_k = poses[k_index].inverse()
    out = [inv_k.compose(g) for g in poses]
    out[k_index] = RigidTransform.identity()
    return out


def rotations_valid(R: np.ndarray) -> np.ndarray:
    """RigidTransform's checks (motion.py:52-62) over stacked (..., 3, 3)
    matrices: allclose(R.T @ R, I, atol=1e-6) and isclose(det R, 1,
    atol=1e-6).  Stacked matmul / det run the same per-matrix kernels as the
    single-matrix calls; entries within 1e-12 of the allclose threshold (or
    non-finite) are re-checked with the per-matrix expression."""
    R = np.asarray(R, np.float64)
    flat = R.reshape(-1, 3, 3)
    eye = np.eye(3)
    with np.errstate(all="ignore"):
        dev = np.abs(np.matmul(np.transpose(flat, (0, 2, 1)), flat) - eye)
        thr = ORTHONORMAL_ATOL + 1e-5 * eye
        orth = np.all(dev <= thr, axis=(1, 2))
        near = np.any(np.abs(dev - thr) < 1e-12, axis=(1, 2)) | ~np.all(np.isfinite(flat), axis=(1, 2))
        detok = np.abs(np.linalg.det(flat) - 1.0) <= ORTHONORMAL_ATOL + 1e-5
    for i in np.flatnonzero(near):
        orth[i] = np.allclose(flat[i].T @ flat[i], eye, atol=ORTHONORMAL_ATOL)
    return (orth & detok).reshape(R.shape[:-2]), orth.reshape(R.shape[:-2])


def poses_to_transform_rows(poses_per_group: Sequence[Sequence], k_index: int) -> np.ndarray:
    """poses_to_transforms + round_f32 for many groups at once, as (G*n, 12)
    rows R | T.  Bit-identical to the per-group path: stacked np.matmul runs
    numpy's per-matrix BLAS kernel for every item (tests/test_host.py pins
    this), and every RigidTransform the per-group path constructs -- input
    poses, the key inverse, the compositions, the float32-rounded results --
    is validated the same way (ValueError on the first invalid one)."""
    G = len(poses_per_group)
    n = len(poses_per_group[0]) if G else 0
    R = np.empty((G, n, 3, 3))
    T = np.empty((G, n, 3))
    for g, poses in enumerate(poses_per_group):
        if len(poses) != n:
            raise ValueError("every group needs the same number of poses")
        for f, p in enumerate(poses):
            if isinstance(p, RigidTransform) or (hasattr(p, "R") and hasattr(p, "T")):
                R[g, f] = np.asarray(p.R, np.float64)
                T[g, f] = np.asarray(p.T, np.float64).reshape(3)
            else:
                Rp, Tp = p
                Rp = np.asarray(Rp, np.float64)
                if Rp.shape != (3, 3):
                    raise ValueError("R must be 3x3")
                R[g, f] = Rp
                T[g, f] = np.asarray(Tp, np.float64).reshape(3)

    def check(M, what):
        ok, orth = rotations_valid(M)
        if not ok.all():
            i = int(np.flatnonzero(~ok.reshape(-1))[0])
            raise ValueError("R is not orthonormal" if not orth.reshape(-1)[i]
                             else "R must be a proper rotation (det +1)")

    check(R, "pose")
    Rk = R[:, k_index]
    Rki = np.transpose(Rk, (0, 2, 1))
    Tki = -np.matmul(Rki, T[:, k_index, :, None])[:, :, 0]
    check(Rki, "inverse")
    CR = np.matmul(Rki[:, None], R)
    CT = np.matmul(Rki[:, None], T[..., None])[..., 0] + Tki[:, None, :]
    check(CR, "compose")
    CR[:, k_index] = np.eye(3)
    CT[:, k_index] = 0.0
    CRf = CR.astype(np.float32).astype(np.float64)
    CTf = CT.astype(np.float32).astype(np.float64)
    check(CRf, "round_f32")
    return np.concatenate([CRf.reshape(G, n, 9), CTf], axis=2).reshape(G * n, 12)


def build_rotation(da: float, db: float, dg: float) -> np.ndarray:
    """Rz(da) @ Ry(db) @ Rx(dg) with the reference's row signs (motion.py:105-116)."""
    ca, sa = np.cos(da), np.sin(da)
    cb, sb = np.cos(db), np.sin(db)
    cg, sg = np.cos(dg), np.sin(dg)
    rz = np.array([[ca, sa, 0.0], [-sa, ca, 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[cb, 0.0, -sb], [0.0, 1.0, 0.0], [sb, 0.0, cb]])
    rx = np.array([[1.0, 0.0, 0.0], [0.0, cg, sg], [0.0, -sg, cg]])
    return rz @ ry @ rx


def integrate_imu(samples: Sequence[ImuSample], t0: float, t1: float, v0=None):
    """Forward-Euler dead reckoning over [t0, t1] with zero-order hold
    (motion.py:119-166): velocity first, then displacement; returns
    (displacement, angles, velocity)."""
    if t1 < t0:
        raise ValueError("t1 must be >= t0")
    v = np.zeros(3) if v0 is None else np.asarray(v0, dtype=np.float64).copy()
    disp = np.zeros(3)
    ang = np.zeros(3)
    if t1 == t0:
        return disp, ang, v
    if not samples:
        raise ImuCoverageError(f"no IMU samples cover [{t0}, {t1}]")
    times = [s.t for s in samples]
    if t0 < times[0] or t1 > times[-1]:
        raise ImuCoverageError(f"IMU span [{times[0]}, {times[-1]}] does not cover [{t0}, {t1}]")
    gaps = np.diff(times)
    nominal = float(np.median(gaps)) if gaps.size else 0.0
    knots = [t0] + times[bisect.bisect_right(times, t0): bisect.bisect_left(times, t1)] + [t1]
    for ta, tb in zip(knots[:-1], knots[1:]):
        dt = tb - ta
        if dt <= 0.0:
            continue
        if nominal > 0.0 and dt > 2.0 * nominal:
            log.warning("IMU gap %.4fs (> 2x nominal %.4fs) at t=%.4f", dt, nominal, ta)
        s = samples[bisect.bisect_right(times, ta) - 1]
        v = v + s.accel * dt
        disp = disp + v * dt
        ang = ang + s.gyro * dt
    return disp, ang, v


def frame_transforms(imu: Sequence[ImuSample], frame_times: Sequence[float],
                     k_index: Optional[int] = None, v0=None) -> List[RigidTransform]:
    """Key-frame alignment from IMU samples (motion.py:169-207)."""
    n = len(frame_times)
    if n == 0:
        return []
    if any(b <= a for a, b in zip(frame_times[:-1], frame_times[1:])):
        raise ValueError("frame_times must be strictly increasing")
    k = n // 2 if k_index is None else k_index
    if not 0 <= k < n:
        raise ValueError("k_index out of range")
    if n == 1:
        return [RigidTransform.identity()]
    steps = []
    v = np.zeros(3) if v0 is None else np.asarray(v0, dtype=np.float64)
    for ta, tb in zip(frame_times[:-1], frame_times[1:]):
        disp, ang, v = integrate_imu(imu, ta, tb, v)
        r = build_rotation(ang[0], ang[1], ang[2])
        steps.append(RigidTransform(r, -(r @ disp)))
    out: List[Optional[RigidTransform]] = [None] * n
    out[k] = RigidTransform.identity()
    for i in range(k - 1, -1, -1):
        out[i] = out[i + 1].compose(steps[i])
    for i in range(k + 1, n):
        out[i] = out[i - 1].compose(steps[i - 1].inverse())
    return out  # type: ignore[return-value]


def ray_trig_tables(w: int, h: int, theta_r: float, phi_r: float, phi_offset: float):
    """sin/cos factors of pixel_ray_grid (range_image.py:141-147), evaluated
    with the same numpy calls so every device-side product
    sin(phi_v) * sin(theta_u) reproduces the reference grid's bits."""
    theta = (np.arange(w, dtype=np.float64) + 0.5) * theta_r
    phi = phi_offset + (np.arange(h, dtype=np.float64) + 0.5) * phi_r
    return (np.ascontiguousarray(np.sin(theta)), np.ascontiguousarray(np.cos(theta)),
            np.ascontiguousarray(np.sin(phi)), np.ascontiguousarray(np.cos(phi)))


def full_scan_width(theta_r: float) -> int:
    return int(round(2.0 * math.pi / theta_r))
