"""B200-native displaced-MPS Gaussian-boson sampler (method "mps").

Public surface mirrors gbsemu (pkg/src/gbsemu/__init__.py:5-63): errors, the
sampler config / batch / entry points, the MPS container and the counter streams.
"""

from .errors import GbsError, NumericalError, ResourceGuardError, ValidationError
from .mps import MPS, SiteShape, bond_dims, device_site, host_site
from .sampler import (
    METHODS,
    MpsSampleBatch,
    MpsSampler,
    MpsSamplerConfig,
    batch_sample,
    chain_joint_probability,
    chain_log_probability,
    sample_one,
)
from .streams import alpha_stream, stream_uniforms

__all__ = [name for name in dir() if not name.startswith("_")]
