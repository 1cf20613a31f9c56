"""S2O prefill attention as a PyTorch operator, for model integration.

    torch.ops.s2o.attention(q, k, v, seg_len, tau, q_reorder, fused) -> o

q [B, Hq, L, D], k/v [B, Hkv, L, D] (GQA when Hkv < Hq; any (batch, head, token) strides with a
unit channel stride, so the transposed projection views of a HuggingFace attention layer go in
without a copy), bf16 or fp32; o has q's shape and dtype, causal softmax scale 1/sqrt(D). The op
is one asynchronous C-ABI call (s2o_attention_fwd) on the current stream: no host
synchronisation, so it can be captured into a CUDA graph; it registers a fake (meta)
implementation for shape propagation. There is no CPU kernel: CPU tensors raise.

`register_transformers()` adds the op to transformers' attention registry as "s2o", so a Llama
model built with attn_implementation="s2o" runs its prefill attention on the B200 kernels.
"""
from __future__ import annotations

import torch

from . import s2o as _s2o

_SCHEMA_DONE = False


@torch.library.custom_op("s2o::attention", mutates_args=())
def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seg_len: int, tau: float,
              q_reorder: bool = True, fused: bool = False) -> torch.Tensor:
    if not q.is_cuda:
        raise RuntimeError("s2o::attention needs CUDA tensors (no CPU fallback)")
    cfg = _s2o.KernelConfig(seg_len=min(seg_len, q.shape[2]), tau=tau, q_reorder=q_reorder and not fused,
                            fused=fused)
    out = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    _s2o.s2o_attention(q, k, v, cfg, out=out, want_plan=False, check=False)
    return out


@attention.register_fake
def _(q, k, v, seg_len, tau, q_reorder=True, fused=False):
    return torch.empty_like(q, memory_format=torch.contiguous_format)


def hf_attention_forward(module, query, key, value, attention_mask, scaling=None, dropout=0.0, **kwargs):
    """transformers attention-interface function (same contract as sdpa_attention_forward):
    query [B, Hq, L, D], key/value [B, Hkv, L, D] -> (output [B, L, Hq, D], None). Prefill only:
    causal, no padding mask, no dropout, scale 1/sqrt(D)."""
    if dropout:
        raise ValueError("s2o attention: dropout is not supported")
    d = query.shape[-1]
    if scaling is not None and abs(float(scaling) - d ** -0.5) > 1e-12:
        raise ValueError("s2o attention computes softmax(q k^T / sqrt(D)); other scalings are not supported")
    if key.shape[2] != query.shape[2]:
        raise ValueError("s2o attention is a prefill operator (query and key lengths must match)")
    cfg = getattr(module.config, "s2o", {}) if hasattr(module, "config") else {}
    out = torch.ops.s2o.attention(query, key, value, int(cfg.get("seg_len", 2048)), float(cfg.get("tau", 0.005)),
                                  bool(cfg.get("q_reorder", True)), bool(cfg.get("fused", False)))
    return out.transpose(1, 2).contiguous(), None


def register_transformers() -> None:
    """Register "s2o" in transformers' AttentionInterface (idempotent)."""
    from transformers import AttentionInterface
    AttentionInterface.register("s2o", hf_attention_forward)
