"""CPU tests of the boundary and host logic: the C-ABI library loads and
exports every symbol include/stpc_b200.h declares; the Python mirror of the
reference API validates like the reference; host-side transforms match the
oracle bit-for-bit; the product refuses to run without a GPU."""

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, gpu_available, load_case
from oracle import oracle


def header_functions():
    src = open(os.path.join(ROOT, "include", "stpc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stpc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2008_06972_b200 import _native

    lib = _native.LIB_PATH
    assert os.path.exists(lib), "build with python -m paper_2008_06972_b200.build"
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(stpc_[a-z0-9_]+)\b", out))
    declared = header_functions()
    assert declared, "header parse failed"
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert sorted(_native.EXPORTS) == declared  # the ctypes binding covers the header


def test_library_is_sm100a():
    from paper_2008_06972_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_loads_and_reports_devices():
    from paper_2008_06972_b200 import _native

    L = _native.load()
    assert L.stpc_version().startswith(b"stpc_b200")
    assert L.stpc_device_count() >= 0


def test_host_scatter_fills_bytes_objects():
    """stpc_host_scatter (host threads, no GPU) behind compress_groups' result
    bytes: every blob lands in its own freshly allocated bytes object,
    including empty blobs and a batch large enough to use several threads."""
    import numpy as np

    from paper_2008_06972_b200 import _native
    from paper_2008_06972_b200.codec import _bytes_from_arena

    L = _native.load()
    rng = np.random.default_rng(5)
    for lens in ([3, 0, 5, 1], [0], list(rng.integers(0, 400_000, 24))):
        lens = np.asarray(lens, np.int64)
        off = np.zeros(len(lens) + 1, np.int64)
        off[1:] = np.cumsum(lens)
        arena = rng.integers(0, 256, int(off[-1]) + 7, dtype=np.uint8)
        got = _bytes_from_arena(L, arena.ctypes.data, off, lens)
        assert [len(b) for b in got] == list(lens)
        for i, b in enumerate(got):
            assert isinstance(b, bytes) and b == arena[off[i]:off[i] + lens[i]].tobytes()


@pytest.mark.skipif(gpu_available(), reason="only meaningful without a GPU")
def test_no_cpu_fallback_without_gpu():
    from paper_2008_06972_b200 import compress, _native

    clouds, poses, cfg, blob, z = load_case("single_4x4")
    with pytest.raises(_native.NativeUnavailable):
        compress(clouds, cfg)


def test_codec_config_validation_mirrors_reference():
    from paper_2008_06972_b200 import CodecConfig

    assert CodecConfig(mode="stream", n_frames=10).k_index == 5
    assert CodecConfig().tau == 0.02 and CodecConfig().w == 1800 and CodecConfig().h == 64
    with pytest.raises(ValueError):
        CodecConfig(mode="bogus")
    with pytest.raises(ValueError):
        CodecConfig(mode="single", n_frames=2)
    with pytest.raises(ValueError):
        CodecConfig(tau=0.0)
    with pytest.raises(ValueError):
        CodecConfig(tile_w=0)
    with pytest.raises(ValueError):
        CodecConfig(mode="stream", n_frames=3, k_index=3)


def test_compress_argument_errors_are_reference_types():
    from paper_2008_06972_b200 import CodecConfig, DataError, compress

    cfg = CodecConfig(mode="stream", n_frames=3)
    with pytest.raises(DataError):
        compress([np.zeros((0, 3), np.float32)] * 2, cfg)  # wrong frame count
    with pytest.raises(DataError):
        compress([np.zeros((0, 3), np.float32)] * 3, cfg)  # stream without poses/IMU


def test_pose_transforms_match_oracle_bits():
    from paper_2008_06972_b200.geometry import poses_to_transforms

    for name in ("stream3_4x4", "stream5_2x2", "stream4_8x4_k0"):
        clouds, poses, cfg, blob, z = load_case(name)
        mine = [t.round_f32() for t in poses_to_transforms(poses, cfg.k_index)]
        ref = oracle.poses_to_transforms(poses, cfg.k_index)
        for t, (R, T) in zip(mine, ref):
            assert np.array_equal(t.R, R) and np.array_equal(t.T, T)


def test_transforms_are_written_into_the_golden_blob():
    """The f32 transform block of the reference blob equals ours (bitstream.py:213-217)."""
    from paper_2008_06972_b200.geometry import poses_to_transforms

    clouds, poses, cfg, blob, z = load_case("stream3_4x4")
    ts = [t.round_f32() for t in poses_to_transforms(poses, cfg.k_index)]
    payload = oracle_payload(blob)
    block = np.frombuffer(payload[57:57 + 48 * cfg.n_frames], "<f4").reshape(cfg.n_frames, 12)
    for t, row in zip(ts, block):
        assert np.array_equal(row.astype(np.float64), t.row12())


def oracle_payload(blob):
    """Decode a blob's entropy stage (test helper: canonical Huffman decode)."""
    lens = np.frombuffer(blob[28:284], np.uint8)
    raw_len = int.from_bytes(blob[8:16], "little")
    codes = oracle.canonical_codes(lens)
    table = {(int(lens[s]), int(codes[s])): s for s in range(256) if lens[s]}
    bits = np.unpackbits(np.frombuffer(blob[284:], np.uint8))
    out = bytearray()
    code = ln = 0
    for bit in bits:
        code = (code << 1) | int(bit)
        ln += 1
        if (ln, code) in table:
            out.append(table[(ln, code)])
            code = ln = 0
            if len(out) == raw_len:
                break
    return bytes(out)


def test_imu_alignment_matches_pose_free_reference_semantics():
    """frame_transforms: key frame is identity, chaining and inversion hold."""
    from paper_2008_06972_b200.geometry import ImuSample, frame_transforms

    imu = [ImuSample(t=0.01 * i, accel=np.array([0.2, 0.0, 0.0]), gyro=np.array([0.0, 0.0, 0.1]))
           for i in range(101)]
    ts = frame_transforms(imu, [0.0, 0.3, 0.6, 0.9], k_index=1)
    assert np.array_equal(ts[1].R, np.eye(3)) and np.array_equal(ts[1].T, np.zeros(3))
    p = np.array([[1.0, 2.0, 3.0]])
    back = ts[2].inverse().apply(ts[2].apply(p))
    assert np.allclose(back, p)


def test_ray_trig_tables_rebuild_reference_grid_bits():
    """sin(phi)*sin(theta) from the tables == pixel_ray_grid's stored values."""
    from paper_2008_06972_b200.geometry import ray_trig_tables

    st, ct, sp, cp = ray_trig_tables(2000, 64, np.pi / 1000, 0.0073, 1.53)
    grid = oracle.ray_grid(2000, 64, np.pi / 1000, 0.0073, 1.53)
    assert np.array_equal(sp[:, None] * st[None, :], grid[:, :, 0])
    assert np.array_equal(sp[:, None] * ct[None, :], grid[:, :, 1])
    assert np.array_equal(np.broadcast_to(cp[:, None], (64, 2000)), grid[:, :, 2])


def test_synthetic_scene_shapes_match_baseline():
    from paper_2008_06972_b200 import synth

    g = synth.make_group(1, 2, synth.SENSOR_64)
    assert all(c.dtype == np.float32 and c.shape[1] == 3 for c in g.clouds)
    assert 115_000 < g.clouds[0].shape[0] < 125_000  # ~120k points (BASELINE configs[0])
    assert len(g.poses) == 2


def _decode_error_cases():
    z = np.load(os.path.join(ROOT, "tests", "golden", "decode_errors.npz"))
    off = z["offsets"]
    return [(str(nm), str(ex), z["blobs"][off[i]:off[i + 1]].tobytes())
            for i, (nm, ex) in enumerate(zip(z["names"], z["expect"]))]


def test_decoder_host_checks_match_reference():
    """The checks the host side of the GPU decoder makes itself -- header
    (bitstream.py:398-409), config block (_parse_config :356-385) and the
    transform block (:420-426) -- raise the reference's exception class on
    the reference-labelled corrupt blobs they decide."""
    import struct

    from oracle import decode as odec
    from paper_2008_06972_b200 import decode

    checked = 0
    for name, expect, blob in _decode_error_cases():
        if name.startswith("hdr_") and name != "hdr_crc":
            with pytest.raises(Exception) as ei:
                decode._header(blob)
            assert type(ei.value).__name__ == expect, name
            checked += 1
        elif name.startswith(("cfg_", "xf_", "trunc_config", "trunc_transforms")):
            raw_len, enc_len = struct.unpack_from("<QQ", blob, 8)
            pl = odec.huffman_decode(np.frombuffer(blob, np.uint8, 256, 28), blob[284:284 + enc_len], raw_len)
            got = "ok"
            try:
                c = decode._config(pl[:57].ljust(57, b"\0"), len(pl))
                decode._transforms(pl[:57 + 48 * c["n_frames"]].ljust(57 + 48 * c["n_frames"], b"\0"), len(pl),
                                   c["n_frames"])
            except Exception as exc:  # noqa: BLE001
                got = type(exc).__name__
            assert got == expect, name
            checked += 1
    assert checked >= 15


def test_decoder_rejects_bad_headers():
    from paper_2008_06972_b200 import MalformedBlobError, TruncatedBlobError, UnknownVersionError
    from paper_2008_06972_b200.decode import _header

    clouds, poses, cfg, blob, z = load_case("single_4x4")
    _header(blob)
    with pytest.raises(TruncatedBlobError):
        _header(blob[:100])
    with pytest.raises(MalformedBlobError):
        _header(b"XXXX" + blob[4:])
    with pytest.raises(UnknownVersionError):
        _header(blob[:4] + b"\x02\x00" + blob[6:])
    with pytest.raises(TruncatedBlobError):
        _header(blob[:-10])


def _imu_of(z):
    from paper_2008_06972_b200 import ImuSample

    return [ImuSample(t=float(t), accel=a, gyro=g) for t, a, g in zip(z["imu_t"], z["imu_accel"], z["imu_gyro"])]


def test_imu_frame_transforms_match_reference_bits():
    """frame_transforms (motion.py:169-207) over a gapped 200 Hz trace equals
    the reference's output bit-for-bit (stored as the fixture's poses)."""
    from paper_2008_06972_b200 import frame_transforms

    clouds, poses, cfg, blob, z = load_case("stream5_imu")
    ts = frame_transforms(_imu_of(z), list(z["frame_times"]), cfg.k_index, z["v0"])
    for t, (R, T) in zip(ts, poses):
        assert np.array_equal(t.R, R) and np.array_equal(t.T, T)


def test_imu_errors_mirror_reference():
    from paper_2008_06972_b200 import ImuCoverageError, frame_transforms, integrate_imu

    clouds, poses, cfg, blob, z = load_case("stream5_imu")
    imu = _imu_of(z)
    with pytest.raises(ImuCoverageError):
        integrate_imu(imu, -1.0, 0.1)
    with pytest.raises(ImuCoverageError):
        integrate_imu([], 0.0, 0.1)
    with pytest.raises(ValueError):
        integrate_imu(imu, 0.2, 0.1)
    with pytest.raises(ValueError):
        frame_transforms(imu, [0.1, 0.1], 0)
    with pytest.raises(ValueError):
        frame_transforms(imu, [0.1, 0.2], 2)
    d, a, v = integrate_imu(imu, 0.1, 0.1, z["v0"])
    assert not d.any() and not a.any() and np.array_equal(v, z["v0"])


def test_decoder_batched_transforms_equal_per_frame_reference_expressions():
    """_transforms_batch (vectorised RigidTransform checks + inverse) gives the
    bits and errors of the per-frame reference expressions (_transforms)."""
    from paper_2008_06972_b200 import decode as D

    rng = np.random.default_rng(3)
    B, n = 64, 8
    heads = np.zeros((B, 57 + 48 * 16), np.uint8)
    for i in range(B):
        q = rng.normal(size=(n, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        w, x, y, z = q.T
        R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                      2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                      2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], 1)
        T = rng.normal(size=(n, 3)) * 30
        heads[i, 57:57 + 48 * n] = np.concatenate([R, T], 1).astype("<f4").view(np.uint8).reshape(-1)
    f32 = lambda v: np.frombuffer(np.float32(v).tobytes(), np.uint8)  # noqa: E731
    heads[5, 57 + 96:57 + 100] = f32(2.0)
    heads[9, 57 + 48 + 36:57 + 48 + 40] = f32(np.nan)
    heads[11, 57 + 144:57 + 148] = f32(np.inf)
    heads[13, 57:57 + 36] = np.diag([1.0, 1.0, -1.0]).reshape(9).astype("<f4").view(np.uint8)
    # scalings whose R^T R diagonal / determinant sit at the tolerances
    # (1e-6 + 1e-5): the native check hands these to the numpy expressions
    for row, target in ((15, 1.1e-5), (17, -1.1e-5), (19, 1.1e-5 / 3), (21, 1.2e-5)):
        s_ = np.float32(np.sqrt(1.0 + target))
        heads[row, 57 + 48:57 + 84] = np.diag([s_, s_, s_]).reshape(9).astype("<f4").view(np.uint8)
    raw_len = np.full(B, 10 ** 6, np.int64)
    raw_len[7] = 100
    good, bad = D._transforms_batch(heads, raw_len, list(range(B)), n)
    assert {5, 7, 11, 13} <= set(bad) and 21 in bad
    for i in range(B):
        try:
            ref = D._transforms(heads[i].tobytes(), int(raw_len[i]), n)
        except Exception as exc:  # noqa: BLE001
            assert type(bad[i]) is type(exc) and str(bad[i]) == str(exc)
            continue
        assert np.array_equal(good[i], ref, equal_nan=True)


def test_batched_pose_transforms_equal_per_group_bits():
    """poses_to_transform_rows (compress_groups' batched path) == per-group
    poses_to_transforms + round_f32, bit for bit, and raises ValueError for an
    invalid pose like the per-group RigidTransform checks."""
    from paper_2008_06972_b200.geometry import RigidTransform, poses_to_transform_rows, poses_to_transforms

    rng = np.random.default_rng(11)
    G, n, k = 40, 8, 3
    groups = []
    for g in range(G):
        q = rng.normal(size=(n, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        w, x, y, z = q.T
        Rs = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                       2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                       2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], 1).reshape(n, 3, 3)
        Ts = rng.normal(size=(n, 3)) * 40
        groups.append([(Rs[i], Ts[i]) if i % 2 else RigidTransform(Rs[i], Ts[i]) for i in range(n)])
    rows = poses_to_transform_rows(groups, k)
    ref = np.concatenate([[t.round_f32().row12() for t in poses_to_transforms(p, k)] for p in groups])
    assert np.array_equal(rows, ref)
    bad = [list(p) for p in groups[:2]]
    bad[1][4] = (np.eye(3) * 2.0, np.zeros(3))
    with pytest.raises(ValueError):
        poses_to_transform_rows(bad, k)


def test_context_pool_bounded_lru_and_exclusive():
    """Encoder/decoder pooling: a checked-out context is never
    handed to a second caller, at most max_idle contexts stay cached, and the
    least recently used config is evicted first."""
    from paper_2008_06972_b200.codec import _checkout, _Pool

    pool = _Pool("STPC_TEST_POOL_UNSET", 2)
    made = []

    def factory(tag):
        def f():
            made.append(tag)
            return object()
        return f

    with _checkout(pool, "a", factory("a")) as a1:
        with _checkout(pool, "a", factory("a")) as a2:
            assert a1 is not a2  # concurrent calls never share a context
    assert made == ["a", "a"]
    with _checkout(pool, "a", factory("a")) as a3:
        assert a3 in (a1, a2)  # reused
    with _checkout(pool, "b", factory("b")):
        pass
    with _checkout(pool, "c", factory("c")):
        pass
    assert sum(len(v) for v in pool.idle.values()) == 2
    assert "a" not in pool.idle  # least recently used config went first
    assert pool.peek("c", factory("c")) is pool.idle["c"][-1]
    pool.clear()
    assert not pool.idle


def test_matmul_contract_probe():
    """The host-BLAS dependence of float64 transforms is detected, not
    assumed: on this build host numpy's pts @ R.T is the
    FMA chain the device and the oracle use (pinned by the stream4_f64
    fixture the reference produced here)."""
    from paper_2008_06972_b200.geometry import matmul_contract

    assert matmul_contract() in ("fma", "plain", "mixed")
    assert matmul_contract() == "fma"
