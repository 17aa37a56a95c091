"""B200-native LJ short-range engine (the hot path of arXiv 2109.10876's taskmd).

The product is libtmd_gpu.so (CUDA C++ for sm_100a behind the C ABI in
include/tmd_gpu.h). This package is the Python mirror of the reference
engine's API on top of it; see engine.py.
"""
from .engine import (  # noqa: F401
    AngleParams, ConfigError, CudaError, Engine, EngineConfig, FeneParams,
    FlatConfig, Interactions, LangevinParams, LjParams, PhysicsError, Section,
    SectionTimers, StateError, StepObservables, VerifyError, counter_normal3,
    counter_uniform3, gen_fcc, thermal_velocities, validate_engine_config,
)
