"""B200-native Cascade-of-Gaussians background subtraction.

Drop-in for the per-pixel hot path of the reference ``cogbg`` package
(arXiv 1705.09339): ``train_engine`` builds the KDE scene prior, pixel
dynamics, mixture warm-up and groups on the GPU; ``CascadeEngine
.process_frame`` runs the fused sm_100a classify+update step and returns
the foreground mask, statistics and per-pixel confidence.  All compute goes
through the C-ABI library ``libcog_b200.so`` (include/cog_b200.h); there is
no CPU fallback.
"""

from .config import EngineConfig, build_config
from .errors import (ClusteringError, CogbgError, ConfigError, CudaError,
                     DataError, FormatError, InternalError, SequenceError,
                     TrainingError, UsageError)
from .frame_io import Frame, FramePlane, LabelMask

__version__ = "0.1.0"

__all__ = [
    "EngineConfig", "build_config", "CogbgError", "ConfigError", "DataError",
    "FormatError", "InternalError", "SequenceError", "UsageError",
    "TrainingError", "ClusteringError", "CudaError", "Frame", "FramePlane",
    "LabelMask", "__version__",
]
