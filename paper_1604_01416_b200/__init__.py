"""dmath_b200: B200-native distributed fp32 GEMM (dMath hot path, arXiv:1604.01416).

The public API mirrors the reference's gridgemm::Session; all work happens in
libdmath_b200.so (tcgen05 fp32-accurate split GEMM, peer-pull panel pipeline, device pool).
"""
from .session import (  # noqa: F401
    Axis, CacheMissError, Config, ConfigError, CudaError, DeadlockError, Error, FillKind, IntegrityError,
    LayoutKind, LayoutSpec, MatrixDescriptor, NcclError, PlanError, Precision, ProtocolError,
    Session, ShapeError, UnsupportedError, UsageError, checkerboard_dims, fill_seeded, local_gemm,
    local_gemm_workspace_size, split_mode_for, presplit_panels,
    make_custom_layout, make_layout, nccl_unique_id, plan_general_gemm, pool_size_class,
)
