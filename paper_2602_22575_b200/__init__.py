"""paper_2602_22575_b200 -- B200-native S2O sparse prefill attention (arxiv 2602.22575).

The product is libs2o_cuda.so (hand-written sm_100a kernels behind the C-ABI in
include/s2o_cuda.h). This package holds its sources (csrc/), the in-tree build
(build.py), a Python mirror of the reference's entry points (s2o.py), head sharding (shard.py),
S2OT tensor files (io.py) and the reference-format benchmark sweep (sweep.py).
"""
from .s2o import (  # noqa: F401
    KernelConfig, TileSpec, SegmentConfig, PermutationPlan, PassBuffers, KernelTrace,
    RankingCost, Representatives, S2oResult, build_plan, build_plan_truncated, segment_representatives,
    pass1_dense_init, pass2_sparse, fused_single_pass, s2o_attention, early_stop_check,
    dense_causal_attention, block_topk_attention, generate_synthetic, attention_host, attention_host_ptr, select_path, lib,
    PATH_AUTO, PATH_GENERIC, PATH_TCGEN05, SCORE_EXACT, SCORE_FAST, S2O_F32, S2O_BF16,
)
