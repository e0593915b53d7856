"""B200-native RKC electro-quasistatic hot path (arXiv 1612.09447).

Drop-in for the reference `eqsim` RKC path: host C++ setup/control + sm_100a
CUDA kernels in libeqs_b200.so behind the C-ABI of include/eqs_b200.h.
"""
from .eqs import (ConfigError, CudaError, EqsError, FemSystem, GeometryError, InvalidArgument, NumericalError,
                  ParseError, PcgResult, StepAttempt, load_library, run_scenario)

__all__ = ["FemSystem", "run_scenario", "load_library", "StepAttempt", "PcgResult", "EqsError", "ConfigError",
           "NumericalError", "GeometryError", "InvalidArgument", "ParseError", "CudaError"]
