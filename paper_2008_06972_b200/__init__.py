"""B200-native compression hot path of the spatio-temporal LiDAR codec of
arXiv 2008.06972, a drop-in for the reference package's ``compress`` path.

Public API (names and meaning follow /root/reference/pkg/src/stpc/__init__.py):

    CodecConfig, EncodeReport, compress, compress_groups, Encoder,
    AngularResolution, RigidTransform, ImuSample, poses_to_transforms,
    frame_transforms, integrate_imu, build_rotation, and the error types.

The compute runs in ``libstpc_b200.so`` (hand-written sm_100a CUDA behind the
C-ABI in include/stpc_b200.h); there is no CPU fallback.
"""

from .codec import (
    MODE_SINGLE,
    MODE_STREAM,
    CodecConfig,
    EncodeReport,
    Encoder,
    TileGrid,
    compress,
    compress_groups,
    get_encoder,
    release_cached,
)
from .decode import DecodeReport, decompress, decompress_full, decompress_many
from .errors import (
    ChecksumError,
    CodecError,
    DataError,
    DecodeError,
    DegenerateFitError,
    ImuCoverageError,
    InsufficientSamplesError,
    MalformedBlobError,
    TruncatedBlobError,
    UnknownVersionError,
)
from .geometry import (
    AngularResolution,
    ImuSample,
    RigidTransform,
    build_rotation,
    frame_transforms,
    integrate_imu,
    poses_to_transforms,
    ray_trig_tables,
)

__version__ = "0.1.0"
