"""Seeded synthetic LiDAR inputs with the BASELINE.json shapes (test/bench harness).

The reference's KITTI evaluation data is not available, so BASELINE.json's
configs are realised here as seeded synthetic scans:

* ground plane z = -1.73 m, ``n_walls`` axis-aligned walls (normals +x, -x,
  +y, -y, repeating) at U(5, 40) m, ``n_boxes`` axis-aligned boxes of size
  U(0.5, 4) m per axis at radius U(3, 50) m and uniform azimuth, resting on
  the ground;
* one ray per pixel centre (the reference's ``cast_frame`` with jitter 0,
  /root/reference/pkg/src/stpc/synth.py:156-231), range noise N(0, sigma)
  applied along the ray, i.i.d. dropouts, cast to float32;
* ego motion of 1.0 m/frame along world +y with 0.5 deg/frame yaw; the poses
  handed to the encoder carry N(0, 0.01 m) translation and N(0, 0.05 deg)
  per-axis rotation noise (frame -> world, the reference's ``poses=``
  convention, /root/reference/pkg/src/stpc/bitstream.py:550-560).

Only the *inputs* come from here; every parity check feeds the identical
float32 arrays to the CUDA path and to the oracle, so the generator's own
floating-point details (torch trig on CPU vs GPU) never enter a comparison.
The generator runs on any torch device; the bench builds its 8192-frame
batch on the GPU in seconds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np
import torch

MIN_RANGE = 0.2
MAX_RANGE = 120.0
GROUND_Z = -1.73


@dataclass(frozen=True)
class Sensor:
    """Spherical range-image geometry (reference CodecConfig fields)."""

    w: int
    h: int
    theta_r: float
    phi_r: float
    phi_offset: float


def _deg(x: float) -> float:
    return x * math.pi / 180.0


# BASELINE.json configs[0..1,3]: 0.18 deg x 0.42 deg, +2.0 .. -24.88 deg.
SENSOR_64 = Sensor(2000, 64, math.pi / 1000.0, _deg(0.42), _deg(88.0))
# configs[2]: 0.1 deg x 0.2 deg; phi_offset 88 deg.
SENSOR_128 = Sensor(3600, 128, _deg(0.1), _deg(0.2), _deg(88.0))
# configs[4]: 0.05 deg x 0.1 deg.
SENSOR_256 = Sensor(7200, 256, _deg(0.05), _deg(0.1), _deg(88.0))

SENSORS = {64: SENSOR_64, 128: SENSOR_128, 256: SENSOR_256}


@dataclass
class SceneSpec:
    walls: List[Tuple[int, float, float]]  # (axis, sign, distance)
    boxes: np.ndarray  # (B, 2, 3) lo/hi corners


def make_scene(rng: np.random.Generator, n_walls: int = 4, n_boxes: int = 20) -> SceneSpec:
    walls = []
    for i in range(n_walls):
        axis = (i // 2) % 2  # x, x, y, y, x, x, ...
        sign = 1.0 if i % 2 == 0 else -1.0
        walls.append((axis, sign, float(rng.uniform(5.0, 40.0))))
    boxes = np.zeros((n_boxes, 2, 3))
    for b in range(n_boxes):
        size = rng.uniform(0.5, 4.0, 3)
        rad = rng.uniform(3.0, 50.0)
        az = rng.uniform(0.0, 2.0 * math.pi)
        cx, cy = rad * math.sin(az), rad * math.cos(az)
        boxes[b, 0] = (cx - size[0] / 2, cy - size[1] / 2, GROUND_Z)
        boxes[b, 1] = (cx + size[0] / 2, cy + size[1] / 2, GROUND_Z + size[2])
    return SceneSpec(walls=walls, boxes=boxes)


def yaw_matrix(psi: float) -> np.ndarray:
    c, s = math.cos(psi), math.sin(psi)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def small_rotation(rx: float, ry: float, rz: float) -> np.ndarray:
    cx, sx = math.cos(rx), math.sin(rx)
    cy, sy = math.cos(ry), math.sin(ry)
    cz, sz = math.cos(rz), math.sin(rz)
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]], dtype=np.float64)
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]], dtype=np.float64)
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]], dtype=np.float64)
    return Rz @ Ry @ Rx


def true_poses(n: int, step_m: float = 1.0, yaw_deg: float = 0.5) -> List[Tuple[np.ndarray, np.ndarray]]:
    return [
        (yaw_matrix(_deg(yaw_deg) * i), np.array([0.0, step_m * i, 0.0]))
        for i in range(n)
    ]


def noisy_poses(rng: np.random.Generator, poses, t_sigma=0.01, r_sigma_deg=0.05):
    out = []
    for R, T in poses:
        dR = small_rotation(*rng.normal(0.0, _deg(r_sigma_deg), 3))
        out.append((dR @ R, T + rng.normal(0.0, t_sigma, 3)))
    return out


def _pixel_dirs(sensor: Sensor, device) -> torch.Tensor:
    u = torch.arange(sensor.w, dtype=torch.float64, device=device)
    v = torch.arange(sensor.h, dtype=torch.float64, device=device)
    theta = (u + 0.5) * sensor.theta_r
    phi = sensor.phi_offset + (v + 0.5) * sensor.phi_r
    sp = torch.sin(phi)[:, None]
    d = torch.stack(
        [sp * torch.sin(theta)[None, :], sp * torch.cos(theta)[None, :],
         torch.cos(phi)[:, None].expand(sensor.h, sensor.w)],
        dim=-1,
    )
    return d.reshape(-1, 3)


def cast_frames(
    scene: SceneSpec,
    poses,
    sensor: Sensor,
    noise: float,
    dropout: float,
    gen: torch.Generator,
    device,
) -> List[torch.Tensor]:
    """Ray-cast every frame of a group; returns float32 (N_i, 3) per frame in
    the frame's own coordinates, pixel raster order, dropouts removed."""
    d_sensor = _pixel_dirs(sensor, device)  # (P, 3)
    boxes = torch.as_tensor(scene.boxes, dtype=torch.float64, device=device)
    out = []
    for R, T in poses:
        Rt = torch.as_tensor(R, dtype=torch.float64, device=device)
        o = torch.as_tensor(T, dtype=torch.float64, device=device)
        d = d_sensor @ Rt.T  # world directions
        best = torch.full((d.shape[0],), math.inf, dtype=torch.float64, device=device)

        def offer(r):
            ok = torch.isfinite(r) & (r > MIN_RANGE) & (r <= MAX_RANGE) & (r < best)
            best.copy_(torch.where(ok, r, best))

        # ground plane z = GROUND_Z
        offer((GROUND_Z - o[2]) / d[:, 2])
        for axis, sign, dist in scene.walls:
            offer((sign * dist - o[axis]) / d[:, axis])
        if boxes.shape[0]:
            inv = 1.0 / d  # (P,3); inf on axis-parallel rays is fine for slabs
            t1 = (boxes[:, None, 0, :] - o) * inv[None]
            t2 = (boxes[:, None, 1, :] - o) * inv[None]
            tn = torch.fmin(t1, t2).amax(dim=-1)
            tf = torch.fmax(t1, t2).amin(dim=-1)
            hit = (tn <= tf) & (tn > MIN_RANGE) & (tn <= MAX_RANGE)
            tn = torch.where(hit, tn, torch.full_like(tn, math.inf))
            offer(tn.amin(dim=0))
        hit = torch.isfinite(best)
        r = best + noise * torch.randn(best.shape, generator=gen, dtype=torch.float64, device=device)
        keep = hit & (torch.rand(best.shape, generator=gen, dtype=torch.float64, device=device) >= dropout) & (r > MIN_RANGE)
        pts = (r[keep, None] * d_sensor[keep]).to(torch.float32)
        out.append(pts)
    return out


@dataclass
class Group:
    """One K+P group: float32 clouds (frame coords) and noisy frame->world poses."""

    clouds: List[np.ndarray]
    poses: List[Tuple[np.ndarray, np.ndarray]]


def make_group(
    seed: int,
    n_frames: int,
    sensor: Sensor = SENSOR_64,
    n_walls: int = 4,
    n_boxes: int = 20,
    noise: float = 0.02,
    dropout: float = 0.05,
    device="cpu",
    as_numpy: bool = True,
):
    """A seeded group (BASELINE configs[1,3] defaults; pass n_walls=8, n_boxes=50,
    noise=0.01, dropout=0.02 and SENSOR_256 for configs[4])."""
    rng = np.random.default_rng(seed)
    scene = make_scene(rng, n_walls, n_boxes)
    poses = true_poses(n_frames)
    enc_poses = noisy_poses(rng, poses) if n_frames > 1 else [(np.eye(3), np.zeros(3))]
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) * 7919 + 17)
    clouds = cast_frames(scene, poses, sensor, noise, dropout, gen, device)
    if as_numpy:
        clouds = [c.cpu().numpy() for c in clouds]
    return Group(clouds=clouds, poses=enc_poses)


def config_params(cfg_id: int):
    """(sensor, n_frames, tile, tau, scene kwargs) for BASELINE.json configs[cfg_id-1]."""
    if cfg_id == 1:
        return SENSOR_64, 1, 4, 0.1, dict()
    if cfg_id == 2:
        return SENSOR_64, 10, 4, 0.1, dict()
    if cfg_id == 3:
        return SENSOR_128, 5, 4, 0.1, dict()
    if cfg_id == 4:
        return SENSOR_64, 8, 4, 0.1, dict()
    if cfg_id == 5:
        return SENSOR_256, 1, 8, 0.05, dict(n_walls=8, n_boxes=50, noise=0.01, dropout=0.02)
    raise ValueError(cfg_id)
