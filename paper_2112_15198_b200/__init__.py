"""paper_2112_15198_b200 -- B200-native IFGF matvec (sm_100a CUDA, FP64).

Drop-in for the reference's operator path (ifgf::apply and friends); see
DESIGN.md and include/ifgf_b200.h.
"""
from .engine import (ApplyReport, DomainError, EngineParams, IFGFError, IFGFRuntimeError,
                     InterpOrders, InvalidArgument, KernelConfig, KernelKind, LevelInfo,
                     LogicError, Plan, PointCloud, StageSeconds, apply, choose_depth,
                     default_params, device_ok, direct_eval, error_at_indices, estimate_error,
                     generate, sample_indices)
from . import configs

__all__ = ["ApplyReport", "DomainError", "EngineParams", "IFGFError", "IFGFRuntimeError",
           "InterpOrders", "InvalidArgument", "KernelConfig", "KernelKind", "LevelInfo",
           "LogicError", "Plan", "PointCloud", "StageSeconds", "apply", "choose_depth",
           "default_params", "device_ok", "direct_eval", "error_at_indices", "estimate_error",
           "generate", "sample_indices", "configs"]
