import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libstpc_b200.so")


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    from oracle import oracle

    oracle.build()


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


def golden_cases():
    return sorted(
        os.path.basename(p)[:-4]
        for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
        if os.path.basename(p) not in ("huffman.npz", "projection.npz", "decode_errors.npz", "decode_overlap.npz")
    )


def load_case(name):
    """(clouds, poses, CodecConfig, blob, npz) of a reference-generated fixture."""
    from paper_2008_06972_b200 import AngularResolution, CodecConfig

    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    n = int(z["n_frames"])
    cfg = CodecConfig(
        mode=str(z["mode"]), tau=float(z["tau"]), tile_w=int(z["tile_w"]), tile_h=int(z["tile_h"]),
        res=AngularResolution(float(z["theta_r"]), float(z["phi_r"])), phi_offset=float(z["phi_offset"]),
        w=int(z["w"]), h=int(z["h"]), n_frames=n, k_index=int(z["k_index"]),
        range_quant=float(z["range_quant"]),
    )
    clouds = [z[f"cloud{i}"] for i in range(n)]
    poses = None
    if "pose_R" in z.files:
        poses = list(zip(z["pose_R"], z["pose_T"]))
    return clouds, poses, cfg, z["blob"].tobytes(), z


def trig_matches_host(z, cfg) -> bool:
    """True when this host's numpy sin/cos reproduce the fixture's trig tables
    (a different libm/SIMD path would change the reference's own output)."""
    theta = (np.arange(cfg.w, dtype=np.float64) + 0.5) * cfg.res.theta_r
    phi = cfg.phi_offset + (np.arange(cfg.h, dtype=np.float64) + 0.5) * cfg.res.phi_r
    mine = np.concatenate([np.sin(theta), np.cos(theta), np.sin(phi), np.cos(phi)])
    return np.array_equal(mine, z["trig"])


def gpu_available() -> bool:
    try:
        from paper_2008_06972_b200 import _native

        return _native.load().stpc_device_count() > 0
    except Exception:
        return False
