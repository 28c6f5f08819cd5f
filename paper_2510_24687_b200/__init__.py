"""B200-native fast 2-D circular-geometry wave operators (arxiv 2510.24687): forward A and
exact adjoint A* behind the C ABI of libtat.so (include/tat.h).  This package is the product
path; it never imports oracle/ (test infrastructure)."""
from .tat import Plan, PlanInfo, TatError, derive, host_multiplier, load_library  # noqa: F401

__all__ = ["Plan", "PlanInfo", "TatError", "derive", "host_multiplier", "load_library"]
