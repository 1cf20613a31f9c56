"""Model integration: the S2O operator as a torch custom op and as a
transformers attention implementation in a (small, random-weight) Llama model.

* torch.ops.s2o.attention equals the C-ABI operator and, at tau = 0 (never stops), dense causal
  SDPA within the bf16 tolerance (max |dO| <= 2.5e-2);
* it is graph-capturable (torch.cuda.graph) with identical replays;
* a 2-layer Llama with head_dim 128 run with attn_implementation="s2o" at tau = 0 matches the
  same model under "sdpa" (relative MSE of the last hidden state <= 1e-3).
"""
from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def test_torch_op_matches_dense_at_tau0_and_captures(cuda):
    torch = cuda
    from paper_2602_22575_b200 import torch_op  # noqa: F401  (registers torch.ops.s2o.attention)
    torch.manual_seed(0)
    q = torch.randn(1, 8, 2048, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, 2, 2048, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, 2, 2048, 128, device="cuda", dtype=torch.bfloat16)
    o = torch.ops.s2o.attention(q, k, v, 512, 0.0, True, False)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    assert (o.float() - ref.float()).abs().max().item() <= 2.5e-2
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        torch.ops.s2o.attention(q, k, v, 512, 0.005, True, False)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        out = torch.ops.s2o.attention(q, k, v, 512, 0.005, True, False)
    g.replay()
    torch.cuda.synchronize()
    eager = torch.ops.s2o.attention(q, k, v, 512, 0.005, True, False)
    assert torch.equal(out, eager)


def test_llama_with_s2o_attention_matches_sdpa_at_tau0(cuda):
    torch = cuda
    transformers = pytest.importorskip("transformers")
    from paper_2602_22575_b200 import torch_op
    torch_op.register_transformers()
    torch.manual_seed(0)
    cfg = transformers.LlamaConfig(hidden_size=1024, num_attention_heads=8, num_key_value_heads=2, head_dim=128,
                                   intermediate_size=2048, num_hidden_layers=2, vocab_size=1000,
                                   max_position_embeddings=4096)
    cfg._attn_implementation = "sdpa"
    model = transformers.LlamaForCausalLM(cfg).to(device="cuda", dtype=torch.bfloat16).eval()
    ids = torch.randint(0, 1000, (1, 2048), device="cuda")
    with torch.no_grad():
        h_dense = model.model(input_ids=ids, use_cache=False).last_hidden_state.float()
        model.config._attn_implementation = "s2o"
        model.config.s2o = {"seg_len": 512, "tau": 0.0}
        for layer in model.model.layers:
            layer.self_attn.config._attn_implementation = "s2o"
        h_s2o = model.model(input_ids=ids, use_cache=False).last_hidden_state.float()
    rel = ((h_s2o - h_dense) ** 2).mean() / (h_dense ** 2).mean()
    assert rel.item() <= 1e-3, rel.item()
