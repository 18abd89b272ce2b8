"""B200-native (sm_100a) SWA decode hot path of ALISA (arXiv 2403.17312).

C ABI: include/skv_b200.h (libskv_b200.so, built from csrc/).
C++ drop-in for the reference `skv` headers: include/skv/b200.hpp.
Python mirror of the reference names: paper_2403_17312_b200.api.
"""
from ._lib import (ContractViolation, CudaError, InfeasiblePlan, OutOfDeviceMemory, Unsupported,
                   build, lib)

__all__ = ["ContractViolation", "CudaError", "InfeasiblePlan", "OutOfDeviceMemory", "Unsupported",
           "build", "lib"]
