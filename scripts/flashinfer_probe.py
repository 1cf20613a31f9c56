"""Dev probe: flashinfer's sm100 prefill as a vendor comparator (best of cuDNN SDPA and
flashinfer) -- the dense causal C3 layer and pass-1's block-diagonal work (segments as a ragged
batch). CUDA events, min of 3. Library code, used only as a comparator."""
import os, sys, time
import torch

L, HQ, HKV, D, S = 131072, 32, 8, 128, 2048
torch.manual_seed(0)
q = torch.randn(L, HQ, D, device="cuda", dtype=torch.bfloat16)
k = torch.randn(L, HKV, D, device="cuda", dtype=torch.bfloat16)
v = torch.randn(L, HKV, D, device="cuda", dtype=torch.bfloat16)


def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best


import flashinfer
out = {}
for backend in ("auto", "cutlass", "fa2"):
    try:
        t0 = time.time()
        ms = t(lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, backend=backend))
        out[f"dense_{backend}"] = ms
        print(f"dense causal C3 backend={backend}: {ms:.3f} ms (first call incl. JIT {time.time() - t0:.0f} s)", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"dense backend={backend}: {type(e).__name__}: {str(e)[:200]}", flush=True)
nseg = L // S
ws = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
indptr = torch.arange(0, L + 1, S, dtype=torch.int32, device="cuda")
for backend in ("auto", "cutlass", "fa2"):
    try:
        w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
        w.plan(indptr, indptr, HQ, HKV, D, causal=True, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        t0 = time.time()
        ms = t(lambda: w.run(q, k, v))
        out[f"blockdiag_{backend}"] = ms
        print(f"block-diagonal ({nseg} x {S}) backend={backend}: {ms:.3f} ms (first call {time.time() - t0:.0f} s)", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"blockdiag backend={backend}: {type(e).__name__}: {str(e)[:200]}", flush=True)
qs = q.view(nseg, S, HQ, D).permute(0, 2, 1, 3)
ks = k.view(nseg, S, HKV, D).permute(0, 2, 1, 3)
vs = v.view(nseg, S, HKV, D).permute(0, 2, 1, 3)
qs, ks, vs = qs.contiguous(), ks.contiguous(), vs.contiguous()
ms = t(lambda: torch.nn.functional.scaled_dot_product_attention(qs, ks, vs, is_causal=True, enable_gqa=True))
print(f"block-diagonal torch SDPA (cuDNN/flash): {ms:.3f} ms", flush=True)
