"""B200-native NanoCP DCP decode-step data path (arXiv 2605.21100).

Product = libdcp_b200.so: hand-written sm_100a kernels behind the C ABI of
include/dcp_capi.h plus the dcpsim C++ drop-in (include/dcpsim/).  This Python
package only binds that ABI for tests and benches (no CPU fallback).
"""
from ._capi import (ConfigError, DcpCudaError, DcpInvalidArgument, DcpUnsupported, EmptyShard,
                    InconsistentPlacement, InsufficientFrames, ShapeOverflow, SimError,
                    UnknownPage, UnknownRequest, lib)

__all__ = ["lib", "SimError", "InsufficientFrames", "UnknownRequest", "UnknownPage",
           "InconsistentPlacement", "ShapeOverflow", "EmptyShard", "ConfigError",
           "DcpInvalidArgument", "DcpUnsupported", "DcpCudaError"]
