"""B200-native fused linear-cross-entropy (SlideFormer §3.3 LCE kernel, arXiv 2603.16428).

Hot path: libslf_lce.so (hand-written sm_100a CUDA: TMA + tcgen05/TMEM GEMM tiles with fused
LCE epilogues) behind the C ABI in include/slf_lce.h; this package is the thin Python binding.
"""
from .lce import (  # noqa: F401
    LCEFunction, LCEFunctionFused, Profile, scale_, alloc_workspace, debug_gemm, dx_finalize, lce_bwd, lce_fwd, lce_fwd_bwd, plan_describe, shard_stats,
    stats_combine, status, workspace_bytes, rmsnorm_fwd, rmsnorm_bwd, rmsnorm_lce_fwd_bwd, SShard, s_plan,
    HostStaging, lce_fwd_bwd_host, Comm, comm_unique_id, lce_fwd_bwd_sharded, sharded_workspace_bytes,
    sharded_plan_describe, sharded_chunk_table, shard_bounds_native, lce_fwd_bwd_dp, target_csr, rmsnorm_lce_workspace_bytes,
    rmsnorm_lce_plan_describe, rmsnorm_workspace_bytes,
)
