"""Llama-3.1-8B-shaped prefill through transformers with the S2O operator as its attention.

    python scripts/llama_prefill.py [--L 131072] [--layers 1] [--tau 0.005] [--graph]

Builds a LlamaForCausalLM with the Llama-3.1-8B layer shape (hidden 4096, 32 q / 8 kv heads,
head_dim 128, MLP 14336, RoPE theta 5e5) and RANDOM weights (no checkpoint is available offline),
runs one prefill forward with attn_implementation="sdpa" (cuDNN/flash) and with "s2o"
(paper_2602_22575_b200.torch_op), and prints one JSON line: ms per forward for both (CUDA events,
after warm-up; optionally a captured CUDA graph for the s2o model), the speedup, and the
relative MSE of the last hidden state. With random weights the attention has no learned structure,
so the sparsity S2O finds here is not that of a trained model (PAPER.md:665-697 reports real
activations); the run demonstrates the integration (custom op, HF attention registry, graph
capture) and the end-to-end time split, not the paper's accuracy numbers.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--tau", type=float, default=0.005)
    ap.add_argument("--seg", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--graph", action="store_true")
    args = ap.parse_args()
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    from paper_2602_22575_b200 import torch_op
    torch_op.register_transformers()
    torch.manual_seed(0)
    cfg = LlamaConfig(hidden_size=4096, num_attention_heads=32, num_key_value_heads=8, head_dim=128,
                      intermediate_size=14336, num_hidden_layers=args.layers, vocab_size=128256,
                      rope_theta=500000.0, max_position_embeddings=max(args.L, 8192), torch_dtype=torch.bfloat16)
    cfg._attn_implementation = "sdpa"
    model = LlamaForCausalLM(cfg).to(device="cuda", dtype=torch.bfloat16).eval()
    ids = torch.randint(0, cfg.vocab_size, (1, args.L), device="cuda")

    def run(impl):
        model.config._attn_implementation = impl
        model.config.s2o = {"seg_len": args.seg, "tau": args.tau}
        for layer in model.model.layers:
            layer.self_attn.config._attn_implementation = impl
        with torch.no_grad():
            return model.model(input_ids=ids, use_cache=False).last_hidden_state

    def timeit(impl):
        run(impl)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(impl)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    dense_ms = timeit("sdpa")
    h_dense = run("sdpa").float()
    s2o_ms = timeit("s2o")
    h_s2o = run("s2o").float()
    rel_mse = float(((h_s2o - h_dense) ** 2).mean() / (h_dense ** 2).mean())
    graph_ms = None
    if args.graph:
        model.config._attn_implementation = "s2o"
        static_out = None
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.no_grad():
            run("s2o")
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g), torch.no_grad():
            static_out = model.model(input_ids=ids, use_cache=False).last_hidden_state
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        graph_ms = a.elapsed_time(b) / args.reps
        assert torch.equal(static_out, run("s2o")), "graph replay differs from eager"
    print(json.dumps({"model": "Llama-3.1-8B layer shape, random weights", "layers": args.layers, "L": args.L,
                      "seg_len": args.seg, "tau": args.tau, "prefill_ms": {"sdpa": round(dense_ms, 2),
                      "s2o": round(s2o_ms, 2), "s2o_cuda_graph": round(graph_ms, 2) if graph_ms else None},
                      "speedup": round(dense_ms / s2o_ms, 3),
                      "last_hidden_rel_mse_vs_sdpa": rel_mse}))


if __name__ == "__main__":
    main()
