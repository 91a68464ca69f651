"""CPU: pin the oracle against fixtures the reference itself produced
(tests/golden/make_golden.py).  No GPU needed."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case, trig_matches_host
from oracle import oracle


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_blob_matches_reference(name):
    clouds, poses, cfg, blob, z = load_case(name)
    if not trig_matches_host(z, cfg):
        pytest.skip("host numpy sin/cos differ from the fixture host's; blob not comparable")
    ob, enc = oracle.compress(clouds, cfg, poses)
    assert ob == blob


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_projection_matches_reference(name):
    clouds, poses, cfg, blob, z = load_case(name)
    ocfg = oracle.OracleConfig.of(cfg)
    ts = oracle.poses_to_transforms(poses, ocfg.k_index) if poses is not None else [(np.eye(3), np.zeros(3))]
    for i, c in enumerate(clouds):
        best, win, counts = oracle.convert(c, *ts[i], ocfg)
        valid = np.isfinite(best)
        ranges = np.where(valid, best, 0.0).reshape(cfg.h, cfg.w)
        assert np.array_equal(ranges, z[f"ranges{i}"])
        assert np.array_equal(win.reshape(cfg.h, cfg.w), z[f"win{i}"].astype(np.int64))
        rej, drop, coll = z[f"counts{i}"]
        assert counts[0] == rej and counts[1] == drop
        assert counts[2] - valid.sum() == coll


def test_oracle_projection_unit_cases():
    z = np.load(os.path.join(GOLDEN, "projection.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in z.files})
    for name in names:
        tr, pr, off, w, h = z[f"{name}_geom"]
        cfg = oracle.OracleConfig("single", 0.1, 4, 4, tr, pr, off, int(w), int(h), 1, 0)
        best, win, counts = oracle.convert(z[f"{name}_pts"], np.eye(3), np.zeros(3), cfg)
        valid = np.isfinite(best)
        assert np.array_equal(np.where(valid, best, 0.0).reshape(int(h), int(w)), z[f"{name}_ranges"]), name
        assert np.array_equal(win.reshape(int(h), int(w)), z[f"{name}_win"]), name
        assert list(counts[:2]) == list(z[f"{name}_counts"][:2]), name
        assert counts[2] - valid.sum() == z[f"{name}_counts"][2], name


def test_oracle_huffman_code_lengths():
    z = np.load(os.path.join(GOLDEN, "huffman.npz"))
    for h, lens, codes in zip(z["hists"], z["lens"], z["codes"]):
        mine = oracle.code_lengths(h)
        assert np.array_equal(mine, lens)
        assert np.array_equal(oracle.canonical_codes(mine), codes)
    assert z["lens"].max() == 32  # the cap-repair path is exercised


def test_oracle_pack_and_crc_known_answer():
    # canonical MSB-first packing of a 2-symbol alphabet and zlib's CRC
    payload = bytes([0, 1, 1, 0, 1, 0, 0, 0, 1])
    blob = oracle.entropy_blob(payload)
    assert blob[:4] == b"STPC"
    lens = np.frombuffer(blob[28:284], np.uint8)
    assert lens[0] == 1 and lens[1] == 1
    # 0->'0', 1->'1': bits 011010001 -> 0x68 0x80
    assert blob[284:] == bytes([0x68, 0x80])


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_decoder_matches_reference_decompress(name):
    """The oracle decoder reproduces stpc.decompress bit-for-bit (sha256 of the
    reference's decoded float64 clouds, stored by make_golden.py)."""
    import hashlib

    from oracle import decode as odec

    clouds, poses, cfg, blob, z = load_case(name)
    if not trig_matches_host(z, cfg):
        pytest.skip("host numpy sin/cos differ from the fixture host's")
    dec = odec.decompress(blob)
    assert [p.shape[0] for p in dec] == list(z["dec_counts"])
    assert [hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in dec] == list(z["dec_sha256"])


def test_oracle_decoder_overlapping_runs_match_reference():
    """decode_overlap.npz: overlapping / duplicated / out-of-order runs that
    the reference's deserialize accepts; the oracle decoder reproduces the
    reference's decompress_full (stream-order last writer, per-(run, pixel)
    failure count)."""
    import hashlib

    from oracle import decode as odec

    z = np.load(os.path.join(GOLDEN, "decode_overlap.npz"))
    from paper_2008_06972_b200 import synth

    sm = synth.Sensor(360, 12, 2 * np.pi / 360, np.radians(2.2), np.radians(88.0))  # make_golden.SMALL
    th = (np.arange(sm.w, dtype=np.float64) + 0.5) * sm.theta_r
    ph = sm.phi_offset + (np.arange(sm.h, dtype=np.float64) + 0.5) * sm.phi_r
    same_trig = np.array_equal(np.concatenate([np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)]), z["trig"])
    for i, name in enumerate(z["names"]):
        blob = z["blobs"][z["offsets"][i]:z["offsets"][i + 1]].tobytes()
        clouds, failed = odec.decompress_full(blob)
        assert [c.shape[0] for c in clouds] == list(z["dec_counts"][i]), name
        assert failed == z["failed"][i], name
        shas = [hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest() for c in clouds]
        if same_trig:
            assert shas == list(z["dec_sha256"][i]), name
