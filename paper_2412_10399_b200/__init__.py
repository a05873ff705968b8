"""B200-native CK-MPM per-substep transfer path (arXiv 2412.10399).

Host-side mirror of the reference's scene/config/material API plus a Python
twin of ``ckmpm::Simulation<T>`` over the sm_100a C-ABI library
``libckmpm_b200.so`` (include/ckmpm_b200.h).  No CPU fallback.
"""
from . import abi  # noqa: F401
from .scene import (ConfigError, DeviceError, InvertedElementError, NumericalError,  # noqa: F401
                    OutOfDomainError, SceneConfig, block_scene, mass_epsilon, seed_particles,
                    to_abi_config)


def Simulation(*args, **kwargs):
    """Construct the device-backed Simulation (loads libckmpm_b200.so)."""
    from .api import Simulation as _S
    return _S(*args, **kwargs)
