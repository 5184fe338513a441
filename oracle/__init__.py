"""CPU oracle for the fused LCE hot path — TEST INFRASTRUCTURE ONLY (see lce_oracle.py)."""
from .lce_oracle import (  # noqa: F401
    MEAN, NONE, SUM, coef_for, combine_shards, lce, lce_output_memory, rmsnorm, rmsnorm_lce, rmsnorm_vjp, rows,
    shard_stats,
)
from .adam_oracle import adam_step, adam_steps, bf16_rne  # noqa: F401,E402
