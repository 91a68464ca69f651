"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference-generated fixtures.  Bit-exact for every integer/byte output;
ranges, plane coefficients and offsets are bit-exact too (fp64 with the
reference's operation order, -fmad=false), so no float tolerance is needed
except for the report-only eps band of CUDA vs glibc trig."""

import ctypes
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case, trig_matches_host
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2008_06972_b200 import _native

    return _native.load(require_device=True)


class Dev:
    """Minimal device buffer through the C-ABI (stpc_malloc / memcpy)."""

    def __init__(self, lib, nbytes):
        self.lib = lib
        self.ptr = ctypes.c_void_p()
        assert lib.stpc_malloc(ctypes.byref(self.ptr), int(nbytes)) == 0
        self.nbytes = int(nbytes)

    @classmethod
    def of(cls, lib, arr):
        arr = np.ascontiguousarray(arr)
        d = cls(lib, max(arr.nbytes, 1))
        if arr.nbytes:
            assert lib.stpc_memcpy_h2d(d.ptr, arr.ctypes.data, arr.nbytes) == 0
        return d

    def get(self, dtype, count):
        out = np.empty(count, dtype)
        assert self.lib.stpc_memcpy_d2h(out.ctypes.data, self.ptr, out.nbytes) == 0
        return out

    def __del__(self):
        self.lib.stpc_free(self.ptr)


def gpu_project(lib, clouds, transforms, w, h, theta_r, phi_r, phi_off, f64=False):
    dt = np.float64 if f64 else np.float32
    pts = np.concatenate([np.asarray(c, dt).reshape(-1, 3) for c in clouds]) if clouds else np.zeros((0, 3), dt)
    off = np.zeros(len(clouds) + 1, np.int64)
    off[1:] = np.cumsum([np.asarray(c).reshape(-1, 3).shape[0] for c in clouds])
    xf = np.stack([np.concatenate([np.asarray(R, np.float64).reshape(9), np.asarray(T, np.float64)])
                   for R, T in transforms])
    F = len(clouds)
    d_pts = Dev.of(lib, pts)
    d_best = Dev(lib, 8 * F * w * h)
    d_win = Dev(lib, 8 * F * w * h)
    counts = np.zeros((F, 3), np.int64)
    rc = lib.stpc_project(d_pts.ptr, int(f64), off.ctypes.data, F, xf.ctypes.data, w, h,
                          theta_r, phi_r, phi_off, d_best.ptr, d_win.ptr, counts.ctypes.data, None)
    assert rc == 0, lib.stpc_last_error()
    return d_best.get(np.float64, F * w * h).reshape(F, -1), d_win.get(np.int64, F * w * h).reshape(F, -1), counts


# --------------------------------------------------------------------------- K1


def test_project_reference_unit_cases(lib):
    z = np.load(os.path.join(GOLDEN, "projection.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in z.files})
    for name in names:
        tr, pr, off, w, h = z[f"{name}_geom"]
        w, h = int(w), int(h)
        best, win, counts = gpu_project(lib, [z[f"{name}_pts"]], [(np.eye(3), np.zeros(3))], w, h, tr, pr, off, f64=True)
        valid = np.isfinite(best[0])
        assert np.array_equal(np.where(valid, best[0], 0.0).reshape(h, w), z[f"{name}_ranges"]), name
        assert np.array_equal(win[0].reshape(h, w), z[f"{name}_win"]), name
        assert list(counts[0, :2]) == list(z[f"{name}_counts"][:2]), name
        assert counts[0, 2] - valid.sum() == z[f"{name}_counts"][2], name


def test_project_empty_cloud(lib):
    best, win, counts = gpu_project(lib, [np.zeros((0, 3), np.float32)], [(np.eye(3), np.zeros(3))], 10, 5, 0.1, 0.1, 0.0)
    assert np.isinf(best).all() and (win == -1).all() and counts.sum() == 0


def test_project_full_size_group_bit_exact(lib):
    """configs[1] shapes: 10 frames, P-frames transformed into the key frame."""
    from paper_2008_06972_b200 import synth

    s = synth.SENSOR_64
    g = synth.make_group(11, 10)
    ocfg = oracle.OracleConfig("stream", 0.1, 4, 4, s.theta_r, s.phi_r, s.phi_offset, s.w, s.h, 10, 5)
    ts = oracle.poses_to_transforms(g.poses, 5)
    best, win, counts = gpu_project(lib, g.clouds, ts, s.w, s.h, s.theta_r, s.phi_r, s.phi_offset)
    for i, c in enumerate(g.clouds):
        ob, ow, oc = oracle.convert(c, *ts[i], ocfg)
        assert np.array_equal(best[i].view(np.uint64), ob.view(np.uint64)), f"frame {i}"
        assert np.array_equal(win[i], ow), f"frame {i}"
        assert np.array_equal(counts[i], oc), f"frame {i}"


def _eps_band(pts, tr, pr, off):
    """Points within 1e-9 (relative) of a bin edge, evaluated with glibc trig
    exactly as the reference bins them."""
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    r = np.sqrt((x * x + y * y) + z * z)
    th = np.arctan2(x, y)
    th = np.where(th < 0, th + 2 * np.pi, th)
    qu = th / tr
    qv = (np.arccos(np.clip(z / r, -1, 1)) - off) / pr
    near = lambda q: np.abs(q - np.rint(q)) <= 1e-9 * np.maximum(1.0, np.abs(q))
    return near(qu) | near(qv)


def test_project_points_on_bin_edges(lib):
    """Points placed exactly on bin edges.  Inside the eps band the GPU bins by
    the correctly rounded angle; glibc's atan2 is not correctly rounded on a
    fraction of such inputs (e.g. atan2(0.13481908443029922,
    0.9592876313549115) is 0.506 ulp off), so pixels may differ there -- and
    only there.  Every difference must trace back to eps-band points."""
    w, h, tr, pr, off = 360, 40, 2 * np.pi / 360, 0.01, 1.3
    th = np.arange(w) * tr
    ph = off + np.arange(h) * pr
    T, Ph = np.meshgrid(th, ph)
    d = np.stack([np.sin(Ph) * np.sin(T), np.sin(Ph) * np.cos(T), np.cos(Ph)], -1).reshape(-1, 3)
    pts = np.concatenate([r * d for r in (1.0, 7.3, 55.5)])
    ocfg = oracle.OracleConfig("single", 0.1, 4, 4, tr, pr, off, w, h, 1, 0)
    ob, ow, oc = oracle.convert(pts, np.eye(3), np.zeros(3), ocfg)
    best, win, counts = gpu_project(lib, [pts], [(np.eye(3), np.zeros(3))], w, h, tr, pr, off, f64=True)
    eps = _eps_band(pts, tr, pr, off)
    diff = np.nonzero(best[0].view(np.uint64) != ob.view(np.uint64))[0]
    for pix in diff:
        g_idx, o_idx = win[0][pix], ow[pix]
        assert (g_idx >= 0 and eps[g_idx]) or (o_idx >= 0 and eps[o_idx]), f"pixel {pix} differs outside the eps band"
    assert counts[0][0] == oc[0]
    print(f"eps-band points {int(eps.sum())}, differing pixels {diff.size}")


def test_project_fine_bins_exact_path_overflow(lib, rng):
    """Bins narrower than the fp32 fast path's margin: every point takes the
    exact fp64 path and the deferral queue overflows into the re-pass."""
    w, h, tr, pr, off = 600000, 3, 2 * np.pi / 600000, 2e-5, np.pi / 2 - 3e-5
    n = 60000
    th = rng.uniform(0, 2 * np.pi, n)
    ph = off + rng.uniform(0, h * pr, n)
    r = rng.uniform(1, 90, n)
    pts = np.stack([r * np.sin(ph) * np.sin(th), r * np.sin(ph) * np.cos(th), r * np.cos(ph)], 1)
    ocfg = oracle.OracleConfig("single", 0.1, 4, 1, tr, pr, off, w, h, 1, 0)
    ob, ow, oc = oracle.convert(pts.astype(np.float32), np.eye(3), np.zeros(3), ocfg)
    best, win, counts = gpu_project(lib, [pts.astype(np.float32)], [(np.eye(3), np.zeros(3))], w, h, tr, pr, off)
    assert np.array_equal(best[0].view(np.uint64), ob.view(np.uint64))
    assert np.array_equal(win[0], ow)
    assert np.array_equal(counts[0], oc)


def _project_at(lib, pts, off, xf, w, h, tr, pr, phi_off, f64, shift):
    """stpc_project with the points `shift` bytes past a 256-aligned
    allocation (shift % 16 != 0 takes the register-staged kernel instead of
    the TMA-staged one)."""
    F = len(off) - 1
    raw = np.ascontiguousarray(pts)
    d = Dev(lib, raw.nbytes + 64)
    dst = ctypes.c_void_p(d.ptr.value + shift)
    if raw.nbytes:
        assert lib.stpc_memcpy_h2d(dst, raw.ctypes.data, raw.nbytes) == 0
    d_best = Dev(lib, 8 * F * w * h)
    d_win = Dev(lib, 8 * F * w * h)
    counts = np.zeros((F, 3), np.int64)
    rc = lib.stpc_project(dst, int(f64), off.ctypes.data, F, xf.ctypes.data, w, h, tr, pr, phi_off,
                          d_best.ptr, d_win.ptr, counts.ctypes.data, None)
    assert rc == 0, lib.stpc_last_error()
    return d_best.get(np.float64, F * w * h).reshape(F, -1), d_win.get(np.int64, F * w * h).reshape(F, -1), counts


@pytest.mark.parametrize("f64", [False, True])
def test_project_staged_and_register_paths(lib, rng, f64):
    """The TMA-staged convert (16-byte aligned points, per-warp cp.async.bulk
    pipelines, the array's unaligned tail loaded directly) and the
    register-staged one (misaligned points) against the oracle: ragged frames
    (including empty ones and frames that end mid-16-byte word), NaN /
    infinite / zero points (rejected by the exact path), out-of-band
    elevations (dropped) and a rotated, translated frame."""
    w, h, tr, pr, phi_off = 500, 16, 2 * np.pi / 500, np.radians(1.68), np.radians(88.0)
    sizes = [0, 1, 2, 3, 255, 256, 257, 4099, 0, 30001, 7]
    clouds = []
    for n in sizes:
        th = rng.uniform(0, 2 * np.pi, n)
        ph = rng.uniform(phi_off - 0.05, phi_off + h * pr + 0.05, n)
        r = rng.uniform(0.5, 80, n)
        c = np.stack([r * np.sin(ph) * np.sin(th), r * np.sin(ph) * np.cos(th), r * np.cos(ph)], 1)
        if n > 10:
            c[rng.integers(0, n, 3)] = np.nan
            c[rng.integers(0, n, 2), 1] = np.inf
            c[rng.integers(0, n, 2)] = 0.0
        clouds.append(c.astype(np.float64 if f64 else np.float32))
    ang = 0.3
    Rz = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1]], np.float32)
    xforms = [(np.eye(3), np.zeros(3)) if i % 2 == 0 else (Rz.astype(np.float64), np.array([1.5, -0.25, 0.125]))
              for i in range(len(clouds))]
    off = np.zeros(len(clouds) + 1, np.int64)
    off[1:] = np.cumsum([c.shape[0] for c in clouds])
    pts = np.concatenate(clouds)
    xf = np.stack([np.concatenate([np.asarray(R, np.float64).reshape(9), np.asarray(T, np.float64)]) for R, T in xforms])
    ocfg = oracle.OracleConfig("single", 0.1, 4, 4, tr, pr, phi_off, w, h, 1, 0)
    ref = [oracle.convert(c, R, T, ocfg) for c, (R, T) in zip(clouds, xforms)]
    for shift in ((0, 16, 8) if f64 else (0, 16, 4, 8)):
        best, win, counts = _project_at(lib, pts, off, xf, w, h, tr, pr, phi_off, f64, shift)
        for f, (ob, ow, oc) in enumerate(ref):
            assert np.array_equal(best[f].view(np.uint64), ob.view(np.uint64)), (shift, f)
            assert np.array_equal(win[f], ow), (shift, f)
            assert np.array_equal(counts[f], oc), (shift, f)
    if f64:  # a double array off its 8-byte alignment is refused, not faulted on
        with pytest.raises(AssertionError, match="aligned"):
            _project_at(lib, pts, off, xf, w, h, tr, pr, phi_off, f64, 4)


@pytest.mark.parametrize("w,h,tr,pr,off", [
    # the reference's own conftest sensor: w=64, h=8 at the default
    # AngularResolution (theta_r = 2 pi / 1800, phi_r = 0.00698, phi_offset
    # 1.48; /root/reference/pkg/tests/conftest.py:14-18) -- the w bins cover
    # 1/28 of the circle, so floor(theta / theta_r) % w wraps ~28 times
    (64, 8, 2 * np.pi / 1800, 0.00698, 1.48),
    # a 90-degree sector sensor (sector_res, conftest.py:27-29)
    (200, 20, np.pi / 2 / 200, 0.5 / 20, 1.2),
    # |phi_offset| too large for the fp32 fast path's float rounding
    (300, 3000, 2 * np.pi / 300, 0.01, -20.0),
])
def test_project_wrapping_sensors(lib, rng, w, h, tr, pr, off):
    """Sensors whose w bins do not span the full circle: the azimuth bin is a
    true modulo (a single subtraction corrupted these pixels)."""
    n = 200_000
    th = rng.uniform(0, 2 * np.pi, n)
    lo, hi = max(0.01, off - 0.05), min(np.pi - 0.01, off + h * pr + 0.05)
    if lo >= hi:
        lo, hi = 0.01, np.pi - 0.01
    ph = rng.uniform(lo, hi, n)
    r = rng.uniform(0.5, 120, n)
    pts = np.stack([r * np.sin(ph) * np.sin(th), r * np.sin(ph) * np.cos(th), r * np.cos(ph)], 1).astype(np.float32)
    ocfg = oracle.OracleConfig("single", 0.1, 4, 4, tr, pr, off, w, h, 1, 0)
    ob, ow, oc = oracle.convert(pts, np.eye(3), np.zeros(3), ocfg)
    best, win, counts = gpu_project(lib, [pts], [(np.eye(3), np.zeros(3))], w, h, tr, pr, off)
    eps = _eps_band(pts.astype(np.float64), tr, pr, off)
    diff = np.nonzero(best[0].view(np.uint64) != ob.view(np.uint64))[0]
    for pix in diff:
        g_idx, o_idx = win[0][pix], ow[pix]
        assert (g_idx >= 0 and eps[g_idx]) or (o_idx >= 0 and eps[o_idx]), f"pixel {pix} differs outside the eps band"
    assert counts[0][0] == oc[0] and counts[0][1] == oc[1]
    assert oc[2] > 0


def test_project_tiny_and_huge_coordinates(lib):
    """Coordinates below 1e-15 or above 1e15 must take the exact fp64 path
    (x = y = 1e-25 underflowed the fp32 elevation)."""
    w, h, tr, pr, off = 360, 180, 2 * np.pi / 360, np.pi / 180, 0.0
    vals = []
    for s in (1e-30, 1e-25, 1e-20, 1e-16, 1e-15, 1e-14, 1e14, 1e15, 1e16):
        for d in ((1, 1, -1), (1, -2, 3), (-3, 1, 0.5), (0.2, 0.1, -7), (1, 0, 0), (0, 1, 1)):
            vals.append(np.array(d) * s)
    pts = np.asarray(vals, np.float64)
    ocfg = oracle.OracleConfig("single", 0.1, 4, 4, tr, pr, off, w, h, 1, 0)
    ob, ow, oc = oracle.convert(pts, np.eye(3), np.zeros(3), ocfg)
    for f64 in (True, False):
        p = pts if f64 else pts.astype(np.float32)
        ob, ow, oc = oracle.convert(p, np.eye(3), np.zeros(3), ocfg)
        best, win, counts = gpu_project(lib, [p], [(np.eye(3), np.zeros(3))], w, h, tr, pr, off, f64=f64)
        assert np.array_equal(best[0].view(np.uint64), ob.view(np.uint64))
        assert np.array_equal(win[0], ow)
        assert np.array_equal(counts[0], oc)


def test_reference_conftest_sensor_blob(rng):
    """The reference test suite's own session config, CodecConfig(mode=
    "stream", n_frames=2, w=64, h=8, default res) -- whole pipeline, blob
    byte-identical to the oracle."""
    from paper_2008_06972_b200 import CodecConfig, compress, synth

    sensor = synth.Sensor(64, 8, 2 * np.pi / 1800, 0.00698, 1.48)
    grp = synth.make_group(31337, 2, sensor, n_boxes=6)
    # plus points in every azimuth: they wrap onto the 64 columns
    clouds = []
    for c in grp.clouds:
        th = rng.uniform(0, 2 * np.pi, 20000)
        ph = 1.48 + rng.uniform(0, 8 * 0.00698, 20000)
        r = rng.uniform(2, 60, 20000)
        extra = np.stack([r * np.sin(ph) * np.sin(th), r * np.sin(ph) * np.cos(th), r * np.cos(ph)], 1)
        clouds.append(np.concatenate([c, extra.astype(np.float32)]))
    cfg = CodecConfig(mode="stream", n_frames=2, w=64, h=8)
    mine, _ = compress(clouds, cfg, poses=grp.poses)
    ref, _ = oracle.compress(clouds, cfg, grp.poses)
    assert mine == ref, _first_divergence(mine, ref)


# ------------------------------------------------------------- whole pipeline


@pytest.mark.parametrize("name", golden_cases())
def test_golden_blob(name):
    from paper_2008_06972_b200 import compress

    clouds, poses, cfg, blob, z = load_case(name)
    mine, rep = compress(clouds, cfg, poses=poses)
    if trig_matches_host(z, cfg):
        assert mine == blob
    else:  # host libm differs from the fixture host: compare with the oracle here
        assert mine == oracle.compress(clouds, cfg, poses)[0]
    if trig_matches_host(z, cfg):
        fr = z["fractions"]
        assert (rep.fractions["temporal"], rep.fractions["spatial"], rep.fractions["residual"]) == tuple(fr)


def test_golden_blob_imu_path():
    """compress(imu_samples=, frame_times=, v0=) == the reference's blob
    (IMU alignment on the host, then the device path)."""
    from paper_2008_06972_b200 import ImuSample, compress

    clouds, poses, cfg, blob, z = load_case("stream5_imu")
    imu = [ImuSample(t=float(t), accel=a, gyro=g) for t, a, g in zip(z["imu_t"], z["imu_accel"], z["imu_gyro"])]
    mine, rep = compress(clouds, cfg, imu_samples=imu, frame_times=list(z["frame_times"]), v0=z["v0"])
    assert mine == (blob if trig_matches_host(z, cfg) else oracle.compress(clouds, cfg, poses)[0])


def _cfg(sensor, n, tau, tile):
    from paper_2008_06972_b200 import AngularResolution, CodecConfig

    return CodecConfig(mode="stream" if n > 1 else "single", tau=tau, tile_w=tile, tile_h=tile,
                       res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                       w=sensor.w, h=sensor.h, n_frames=n)


def _first_divergence(a: bytes, b: bytes) -> str:
    n = min(len(a), len(b))
    d = next((i for i in range(n) if a[i] != b[i]), n)
    return f"len {len(a)} vs {len(b)}, first differing byte {d}"


@pytest.mark.parametrize("cfg_id", [1, 2, 5])
def test_baseline_config_blob_full_size(cfg_id):
    """BASELINE.json configs[0], [1], [4] at full size: blob byte-identical."""
    from paper_2008_06972_b200 import compress, synth

    sensor, n, tile, tau, scene = synth.config_params(cfg_id)
    g = synth.make_group(1000 + cfg_id, n, sensor, **scene)
    cfg = _cfg(sensor, n, tau, tile)
    mine, rep = compress(g.clouds, cfg, poses=g.poses if n > 1 else None)
    ref, enc = oracle.compress(g.clouds, cfg, g.poses if n > 1 else None)
    assert mine == ref, _first_divergence(mine, ref)
    for ch, cov in enumerate(rep.coverage):
        assert cov["temporal"] + cov["fallback"] + cov["residual"] == cov["valid"]
        assert cov["valid"] == int(enc.valid[ch].sum())
        assert cov["residual"] == enc.residual_flat[ch].size


@pytest.mark.parametrize("tile,tau", [(2, 0.2), (4, 0.05), (8, 0.1), (16, 0.02)])
def test_config3_sweep_points(tile, tau):
    """BASELINE.json configs[2] (128-beam, 1K+4P) sweep corners."""
    from paper_2008_06972_b200 import compress, synth

    g = synth.make_group(3000 + tile, 5, synth.SENSOR_128)
    cfg = _cfg(synth.SENSOR_128, 5, tau, tile)
    mine, _ = compress(g.clouds, cfg, poses=g.poses)
    ref, _ = oracle.compress(g.clouds, cfg, g.poses)
    assert mine == ref, _first_divergence(mine, ref)


def test_batch_equals_per_group():
    """configs[3] shape: independent 1K+7P groups in one device pass."""
    from paper_2008_06972_b200 import compress, compress_groups, synth

    cfg = _cfg(synth.SENSOR_64, 8, 0.1, 4)
    groups = [synth.make_group(4000 + i, 8) for i in range(3)]
    blobs, reps = compress_groups([g.clouds for g in groups], cfg, [g.poses for g in groups])
    for g, b in zip(groups, blobs):
        assert b == oracle.compress(g.clouds, cfg, g.poses)[0]
        assert b == compress(g.clouds, cfg, poses=g.poses)[0]


@pytest.mark.parametrize("G,f64", [(70, False), (131, False), (66, True)])
def test_compress_groups_gather_pipeline(G, f64):
    """compress_groups hands per-frame arrays to stpc_encode_host_gather
    (threaded gather into pinned staging, pipelined in 8 / 16 chunks, blobs
    in the encoder's own arena, grown on demand); every blob equals the
    single-group compress, and spot checks equal the oracle.  Includes empty
    frames and a float64 batch."""
    import math

    from paper_2008_06972_b200 import AngularResolution, CodecConfig, compress, compress_groups, synth

    sensor = synth.Sensor(300, 12, 2 * math.pi / 300, math.radians(2.0), math.radians(88.0))
    cfg = CodecConfig(mode="stream", tau=0.1, tile_w=4, tile_h=3,
                      res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                      w=sensor.w, h=sensor.h, n_frames=3)
    groups, poses = [], []
    for gi in range(G):
        grp = synth.make_group(8000 + gi, 3, sensor, n_boxes=4)
        clouds = [c.astype(np.float64) for c in grp.clouds] if f64 else list(grp.clouds)
        if gi % 17 == 5:
            clouds[1] = np.zeros((0, 3), clouds[1].dtype)  # an empty frame
        groups.append(clouds)
        poses.append(grp.poses)
    blobs, reps = compress_groups(groups, cfg, poses)
    assert len(blobs) == G
    for gi in (0, 5, G // 2, G - 1):
        assert blobs[gi] == compress(groups[gi], cfg, poses=poses[gi])[0]
        assert blobs[gi] == oracle.compress(groups[gi], cfg, poses[gi])[0]
    assert sum(reps[5].point_counts) == sum(c.shape[0] for c in groups[5])


def test_fit_intermediates_match_oracle():
    """Runs (s, len, f32 a/b/c), temporal offsets and tile classes per chain."""
    from paper_2008_06972_b200 import _native, get_encoder, compress, synth

    sensor = synth.SENSOR_64
    cfg = _cfg(sensor, 4, 0.1, 4)
    g = synth.make_group(77, 4)
    compress(g.clouds, cfg, poses=g.poses)
    enc = get_encoder(cfg)
    ref, oe = oracle.compress(g.clouds, cfg, g.poses)
    tx, ty = cfg.grid().tiles_x, cfg.grid().tiles_y
    n, k = 4, cfg.k_index
    n_runs = enc.copy_buffer(_native.BUF_N_RUNS, np.int32, n * ty).reshape(n, ty)
    rs = enc.copy_buffer(_native.BUF_RUN_S, np.uint16, n * ty * tx).reshape(n, ty, tx)
    rl = enc.copy_buffer(_native.BUF_RUN_LEN, np.uint16, n * ty * tx).reshape(n, ty, tx)
    abc = enc.copy_buffer(_native.BUF_RUN_ABC, np.float32, n * ty * tx * 3).reshape(n, ty, tx, 3)
    # key frame runs
    j = 0
    for tr in range(ty):
        m = n_runs[k, tr]
        sel = oe.t_row == tr
        assert m == sel.sum(), f"tile-row {tr}"
        assert np.array_equal(rs[k, tr, :m], oe.t_s[sel])
        assert np.array_equal(rl[k, tr, :m], oe.t_len[sel])
        assert np.array_equal(abc[k, tr, :m].astype(np.float64), oe.t_abc[sel])
        j += m
    # fallback runs of P frames
    for ch in range(n):
        if ch == k:
            continue
        rows = {tr: (s, ln, a) for tr, s, ln, a in oe.fallback[ch]}
        for tr in range(ty):
            m = n_runs[ch, tr]
            if tr not in rows:
                assert m == 0
                continue
            s, ln, a = rows[tr]
            assert m == s.size
            assert np.array_equal(rs[ch, tr, :m], s) and np.array_equal(rl[ch, tr, :m], ln)
            assert np.array_equal(abc[ch, tr, :m].astype(np.float64), a)


@pytest.mark.parametrize("G", [70, 131])
def test_pipelined_host_encode_matches_device_path(G):
    """stpc_encode_host with >= 64 groups overlaps H2D with compute in 8
    chunks (16 from 128 groups; 131 leaves a short and an empty chunk);
    every blob and frame statistic must equal the one-shot result."""
    import math

    from paper_2008_06972_b200 import AngularResolution, CodecConfig, Encoder, synth

    sensor = synth.Sensor(400, 16, 2 * math.pi / 400, math.radians(1.68), math.radians(88.0))
    cfg = CodecConfig(mode="stream", tau=0.1, tile_w=4, tile_h=4,
                      res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                      w=sensor.w, h=sensor.h, n_frames=3)
    from paper_2008_06972_b200.geometry import poses_to_transforms

    clouds, xf = [], []
    for gi in range(G):
        grp = synth.make_group(500 + gi, 3, sensor, n_boxes=5)
        clouds.extend(grp.clouds)
        xf.extend(t.round_f32().row12() for t in poses_to_transforms(grp.poses, 1))
    pts = np.ascontiguousarray(np.concatenate(clouds))
    off = np.zeros(len(clouds) + 1, np.int64)
    off[1:] = np.cumsum([c.shape[0] for c in clouds])
    xf = np.asarray(xf)
    enc = Encoder(cfg)
    enc.encode_host(G, pts, off, xf)  # one-shot (no output buffer -> not pipelined)
    ref_blobs = enc.blobs()
    ref_stats = enc.frame_stats()
    out = np.zeros(sum(len(b) + 16 for b in ref_blobs) + 4096, np.uint8)
    enc.encode_host(G, pts, off, xf, out)  # pipelined
    o, ln = enc.blob_layout()
    assert [out[a:a + n].tobytes() for a, n in zip(o[:-1], ln)] == ref_blobs
    assert np.array_equal(enc.frame_stats(), ref_stats)
    # spot-check against the oracle
    ocfg_poses = None
    assert ref_blobs[5] == oracle.compress(clouds[15:18], cfg, synth.make_group(505, 3, sensor, n_boxes=5).poses)[0]


def _odd_sensor():
    import math

    from paper_2008_06972_b200 import synth

    return synth.Sensor(333, 13, 2 * math.pi / 333, math.radians(2.1), math.radians(87.0))


@pytest.mark.parametrize(
    "n,k,tile,tau,scale,mutate",
    [
        (12, None, (4, 4), 0.1, 1.0, None),   # 2-byte presence masks
        (3, 0, (3, 3), 0.05, 1.0, None),      # key frame first, 9-pixel tiles
        (4, 3, (5, 2), 0.2, 1.0, None),       # key frame last, non-square tiles
        (3, None, (4, 4), 0.1, 20.0, None),   # ranges past u16 quantisation -> escapes, r_max
        (3, None, (2, 2), 1e-6, 1.0, None),   # everything residual
        (3, None, (4, 4), 0.1, 1.0, "nan"),   # one frame with no valid points
    ],
)
def test_edge_cases_blob(n, k, tile, tau, scale, mutate):
    from paper_2008_06972_b200 import AngularResolution, CodecConfig, compress, synth

    sensor = _odd_sensor()
    grp = synth.make_group(900 + n + tile[0], n, sensor, n_boxes=8)
    clouds = [c * np.float32(scale) for c in grp.clouds]
    if mutate == "nan":
        clouds[0] = np.full_like(clouds[0], np.nan)
    cfg = CodecConfig(mode="stream", tau=tau, tile_w=tile[0], tile_h=tile[1],
                      res=AngularResolution(sensor.theta_r, sensor.phi_r), phi_offset=sensor.phi_offset,
                      w=sensor.w, h=sensor.h, n_frames=n, k_index=k)
    mine, rep = compress(clouds, cfg, poses=grp.poses)
    ref, enc = oracle.compress(clouds, cfg, grp.poses)
    assert mine == ref, _first_divergence(mine, ref)
    for ch, cov in enumerate(rep.coverage):
        assert cov["temporal"] + cov["fallback"] + cov["residual"] == cov["valid"]
    if scale > 1:
        q = np.concatenate([np.rint(r / cfg.range_quant) for r in enc.residual_r])
        assert (q >= 0xFFFF).any()  # the escape path was exercised


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_small_configs_blob(seed):
    """Seeded random small configurations -- odd sensor sizes and resolutions,
    tiles from 1x1 to 7x6 (both fit kernels), k anywhere, 1..12 frames, tau
    from tight to loose, coarse and fine quantisation, float64 clouds -- GPU
    blob == oracle blob byte for byte, and the GPU decoder inverts it exactly
    like the oracle decoder."""
    from oracle import decode as odec
    from paper_2008_06972_b200 import AngularResolution, CodecConfig, compress, decompress, synth

    rng = np.random.default_rng(7000 + seed)
    w = int(rng.integers(40, 400))
    h = int(rng.integers(4, 40))
    sensor = synth.Sensor(w, h, 2 * np.pi / w * float(rng.uniform(0.5, 1.0)), float(rng.uniform(0.01, 0.06)),
                          float(rng.uniform(1.2, 1.7)))
    n = int(rng.integers(1, 13))
    tw, th = int(rng.integers(1, 8)), int(rng.integers(1, 7))
    tau = float(rng.choice([0.005, 0.02, 0.1, 0.3, 1.0]))
    quant = float(rng.choice([0.001, 0.0005, 0.01, 0.05]))
    grp = synth.make_group(7100 + seed, n, sensor, n_boxes=int(rng.integers(2, 30)),
                           noise=float(rng.uniform(0.0, 0.05)), dropout=float(rng.uniform(0.0, 0.3)))
    clouds = list(grp.clouds)
    if seed % 4 == 3:
        clouds = [c.astype(np.float64) * (1.0 + 1e-7) for c in clouds]
    mode = "single" if n == 1 else "stream"
    k = None if n == 1 else int(rng.integers(0, n))
    cfg = CodecConfig(mode=mode, tau=tau, tile_w=tw, tile_h=th, res=AngularResolution(sensor.theta_r, sensor.phi_r),
                      phi_offset=sensor.phi_offset, w=sensor.w, h=sensor.h, n_frames=n, k_index=k,
                      range_quant=quant)
    poses = grp.poses if n > 1 else None
    mine, rep = compress(clouds, cfg, poses=poses)
    ref, _ = oracle.compress(clouds, cfg, poses)
    assert mine == ref, (seed, _first_divergence(mine, ref))
    for a, b in zip(decompress(mine), odec.decompress(mine)):
        assert np.array_equal(a, b)


def test_single_mode_f64_input_full_size():
    """configs[0] through the float64 input path (reference up-casts to f64)."""
    from paper_2008_06972_b200 import compress, synth

    sensor, n, tile, tau, scene = synth.config_params(1)
    g = synth.make_group(77, 1, sensor)
    clouds = [g.clouds[0].astype(np.float64) * 1.0000001]  # not f32-representable
    cfg = _cfg(sensor, 1, tau, tile)
    mine, _ = compress(clouds, cfg)
    assert mine == oracle.compress(clouds, cfg)[0]


# ------------------------------------------------------------------- decoder


@pytest.mark.parametrize("name", golden_cases())
def test_decompress_golden_matches_reference(name):
    """GPU decompress == reference stpc.decompress (sha256 of the exact float64
    clouds the reference produced for this fixture)."""
    import hashlib

    from oracle import decode as odec
    from paper_2008_06972_b200 import decompress

    clouds, poses, cfg, blob, z = load_case(name)
    mine = decompress(blob)
    ref = odec.decompress(blob)
    assert [p.shape for p in mine] == [p.shape for p in ref]
    for a, b in zip(mine, ref):
        assert np.array_equal(a, b)
    if trig_matches_host(z, cfg):
        assert [hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in mine] == list(z["dec_sha256"])


@pytest.mark.parametrize("cfg_id", [2, 3])
def test_decompress_full_size_roundtrip(cfg_id):
    """configs[1] / configs[2]: compress on the GPU, decompress on the GPU,
    bit-identical to the oracle decoder; decoded ranges within tau of the
    input range image on plane pixels and exact (pre-quantisation) otherwise."""
    from oracle import decode as odec
    from paper_2008_06972_b200 import compress, decompress_full, synth

    sensor, n, tile, tau, scene = synth.config_params(cfg_id)
    g = synth.make_group(2000 + cfg_id, n, sensor, **scene)
    cfg = _cfg(sensor, n, tau, tile)
    blob, rep = compress(g.clouds, cfg, poses=g.poses)
    mine, drep = decompress_full(blob)
    ref = odec.decompress(blob)
    for a, b in zip(mine, ref):
        assert a.shape == b.shape and np.array_equal(a, b)
    assert sum(drep.point_counts) == sum(p.shape[0] for p in ref)


def test_decompress_many_batch_and_corruption():
    from paper_2008_06972_b200 import ChecksumError, DecodeError, compress_groups, decompress_many, synth
    from oracle import decode as odec

    cfg = _cfg(synth.SENSOR_64, 3, 0.1, 4)
    groups = [synth.make_group(5000 + i, 3) for i in range(3)]
    blobs, _ = compress_groups([g.clouds for g in groups], cfg, [g.poses for g in groups])
    clouds, reps = decompress_many(blobs)
    for b, cl in zip(blobs, clouds):
        for a, r in zip(cl, odec.decompress(b)):
            assert np.array_equal(a, r)
    bad = bytearray(blobs[0])
    bad[400] ^= 0x55
    with pytest.raises(ChecksumError):
        decompress_many([bytes(bad)])
    with pytest.raises(DecodeError):
        decompress_many([blobs[0][:-3]])


def test_decode_errors_match_reference():
    """Corrupt blobs (tests/golden/decode_errors.npz, labelled by the
    reference's own decompress): the GPU decoder raises the same exception
    class, including which of two errors comes first in reading order; the
    valid ones decode bit-identically to the oracle decoder."""
    from conftest import ROOT
    from oracle import decode as odec
    from paper_2008_06972_b200 import decompress

    z = np.load(os.path.join(ROOT, "tests", "golden", "decode_errors.npz"))
    off = z["offsets"]
    bad = []
    for i, (name, expect) in enumerate(zip(z["names"], z["expect"])):
        blob = z["blobs"][off[i]:off[i + 1]].tobytes()
        try:
            out = decompress(blob)
            got = "ok"
        except Exception as exc:  # noqa: BLE001
            got = type(exc).__name__
        if got != str(expect):
            bad.append((str(name), str(expect), got))
            continue
        if got == "ok":
            for a, b in zip(out, odec.decompress(blob)):
                assert np.array_equal(a, b, equal_nan=True), name
    assert not bad, bad


def test_decompress_many_mixed_batch_reports_first_error():
    """A batch with a corrupt blob in the middle raises that blob's error;
    the same blobs without it decode like one-at-a-time calls."""
    from conftest import ROOT
    from paper_2008_06972_b200 import MalformedBlobError, decompress, decompress_many

    z = np.load(os.path.join(ROOT, "tests", "golden", "decode_errors.npz"))
    off = z["offsets"]
    blobs = {str(nm): z["blobs"][off[i]:off[i + 1]].tobytes() for i, nm in enumerate(z["names"])}
    good = [load_case(n)[3] for n in ("stream3_4x4", "single_4x4", "stream5_2x2", "stream3_4x4")]
    with pytest.raises(MalformedBlobError):
        decompress_many(good[:2] + [blobs["run_len0"]] + good[2:])
    clouds, reps = decompress_many(good)
    for b, cl in zip(good, clouds):
        for a, r in zip(cl, decompress(b)):
            assert np.array_equal(a, r)


def test_repeated_calls_deterministic_and_coverage_partition():
    """Reference acceptance 5 and 9 (pkg/tests/test_acceptance.py:224-251,
    343-368): the same input gives the same bytes on every call (the encoder
    reuses its workspace and alternates its double-buffered range grids), and
    every frame's valid pixels split exactly into temporal + spatial fallback +
    residual (temporal.py:258-290)."""
    from paper_2008_06972_b200 import compress_groups, synth

    cfg = _cfg(synth.SENSOR_64, 10, 0.1, 4)  # configs[1] shape
    groups = [synth.make_group(6100 + i, 10) for i in range(2)]
    clouds, poses = [g.clouds for g in groups], [g.poses for g in groups]
    first, reps = compress_groups(clouds, cfg, poses)
    for _ in range(3):
        again, _ = compress_groups(clouds, cfg, poses)
        assert again == first
    for rep in reps:
        assert len(rep.coverage) == cfg.n_frames
        for c in rep.coverage:
            assert c["temporal"] + c["fallback"] + c["residual"] == c["valid"]
        # the key frame's runs carry its own offset, so they count as temporal
        # (coverage_counts, temporal.py:269-290); it has no fallback rows
        assert rep.coverage[cfg.k_index]["fallback"] == 0
        assert rep.coverage[cfg.k_index]["temporal"] > 0
        assert sum(c["temporal"] for i, c in enumerate(rep.coverage) if i != cfg.k_index) > 0


def test_decompress_overlapping_runs_match_reference():
    """Blobs with overlapping temporal runs, a failing overlap, reversed run
    order, and duplicated / overlapping fallback runs (decode_overlap.npz,
    made by the reference's own serialize): the GPU decoder replays the
    reference's stream-order semantics -- last successful reconstruction
    wins, failures count per (run, pixel) (temporal.py:307-331) -- and its
    clouds and failure count equal the reference's decompress_full."""
    import hashlib

    from oracle import decode as odec
    from paper_2008_06972_b200 import decompress_full, decompress_many

    z = np.load(os.path.join(GOLDEN, "decode_overlap.npz"))
    from paper_2008_06972_b200 import synth

    sm = synth.Sensor(360, 12, 2 * np.pi / 360, np.radians(2.2), np.radians(88.0))
    th = (np.arange(sm.w, dtype=np.float64) + 0.5) * sm.theta_r
    ph = sm.phi_offset + (np.arange(sm.h, dtype=np.float64) + 0.5) * sm.phi_r
    same_trig = np.array_equal(np.concatenate([np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)]), z["trig"])
    blobs = []
    for i, name in enumerate(z["names"]):
        blob = z["blobs"][z["offsets"][i]:z["offsets"][i + 1]].tobytes()
        blobs.append(blob)
        clouds, rep = decompress_full(blob)
        ref, ref_failed = odec.decompress_full(blob)
        for a, b in zip(clouds, ref):
            assert np.array_equal(a, b), name
        assert rep.failed_reconstructions == ref_failed == z["failed"][i], name
        if same_trig:
            assert [hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest() for c in clouds] == \
                list(z["dec_sha256"][i]), name
    # mixed in one batch with ordinary blobs (only the flagged ones take the ordered path)
    good = load_case("stream3_4x4")[3]
    clouds, reps = decompress_many([good] + blobs + [good])
    assert [r.failed_reconstructions for r in reps[1:-1]] == list(z["failed"])
    for a, b in zip(clouds[0], odec.decompress(good)):
        assert np.array_equal(a, b)


def test_entropy_stage_cap_repair_on_device(lib):
    """The device entropy stage (stpc_entropy_encode: histogram, code lengths,
    canonical codes, packing, CRC) on payloads with Fibonacci byte counts:
    34 symbols give a 33-deep Huffman tree, so the 32-bit cap repair
    (huffman.py:51-58; entropy.cu code_lengths_kernel) must run.  Blobs equal
    the oracle's byte for byte (the oracle's code lengths are pinned against
    the reference's on huffman.npz's 40-symbol Fibonacci case)."""
    rng = np.random.default_rng(11)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    payloads = []
    for nsym, perm in ((34, False), (35, True), (33, False)):
        h = np.zeros(256, np.int64)
        syms = rng.permutation(256)[:nsym] if perm else np.arange(nsym)
        h[syms] = fib[:nsym]
        p = np.repeat(np.arange(256, dtype=np.uint8), h)
        rng.shuffle(p)
        payloads.append(p.tobytes())
        assert oracle.code_lengths(h).max() == 32 and (nsym < 34 or nsym - 1 > 32)
    payloads += [bytes([9]) * 1000, b"", bytes(rng.integers(0, 256, 5000, dtype=np.uint8))]
    buf = np.frombuffer(b"".join(payloads), np.uint8)
    off = np.zeros(len(payloads) + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in payloads])
    cap = sum(len(p) for p in payloads) + 300 * len(payloads) + 4096
    out = np.zeros(cap, np.uint8)
    oo = np.zeros(len(payloads) + 1, np.int64)
    rc = lib.stpc_entropy_encode(buf.ctypes.data, off.ctypes.data, len(payloads), out.ctypes.data, cap, oo.ctypes.data)
    assert rc == 0, lib.stpc_last_error()
    for i, p in enumerate(payloads):
        mine = out[oo[i]:oo[i + 1]].tobytes()
        ref = oracle.entropy_blob(p)
        assert mine == ref, (i, _first_divergence(mine, ref))
    assert out[oo[0] + 28:oo[0] + 284].max() == 32  # the repaired table reached the cap
