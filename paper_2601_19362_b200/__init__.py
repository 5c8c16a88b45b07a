"""B200-native On-Demand Communication (ODC) hot path (arXiv 2601.19362).

The ODC path — block shard layout, fetch (gather), push (scatter-accumulate),
the once-per-minibatch barrier, fused AdamW and the LB-Mini load balancer —
runs in libodc.so (hand-written sm_100a kernels + host C++ behind the C ABI of
include/odc/odc.h). This package is the Python host mirror of the
reference's interface (primitives, partition) plus the multi-GPU engine.
"""
from . import errors
from .errors import (BarrierTimeout, DeviceError, InfeasibleError, InvariantError, ModeError, ParamError,
                     ProtocolError, RangeError, StateError)

__all__ = ["errors", "ParamError", "InfeasibleError", "InvariantError", "ProtocolError", "StateError", "ModeError",
           "DeviceError", "BarrierTimeout", "RangeError"]
