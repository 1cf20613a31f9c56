"""Regenerate tests/golden/*.npz from the compiled reference (oracle/_ref/libs2o_ref.so).

    python tests/golden/make_golden.py

Run in the build container (it needs /root/reference to build the reference .so; the
fixtures it writes are committed and read by the tests everywhere, including the GPU
box). Inputs are NOT stored: they are regenerated bit-exactly from their synthetic spec
(generate_synthetic, proj/src/synthetic.cpp:276-328) by the reference generator, which
tests/test_synthetic.py proves identical to the product's host generator.

Fixtures
  c1_golden.npz   C1 = BASELINE.json configs[0]: 1 head, L=4096, D=128, fp32, S=512,
                  tiles 64x64, tau=0.005, mixed stripes (L/64), gain 8, seed 0.
  gqa_golden.npz  small Llama-shaped GQA case on bf16-rounded inputs: Hq=4, Hkv=2, L=4096,
                  D=128, S=512, tiles 128x128, tau=0.005, K/V expanded h -> h/2 for the
                  reference (which has no GQA).
Each stores the reference's plan (q_perm, kv_perm), trace (processed, pair counts),
every 8th output row, a SHA-256 of the full fp32 output, and MSE/MAE/sparsity against
the reference's own dense_causal_attention.
"""
from __future__ import annotations

import hashlib
import os
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, build  # noqa: E402


@dataclass
class Cfg:
    seg_len: int
    tau: float
    b_m: int
    b_n: int
    q_reorder: bool = True
    fused: bool = False
    local_window: int = -1


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) -> fp32, as torch does."""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def c1_inputs(ref: Ref):
    return ref.generate_synthetic("mixed", 4096 // 64, 8.0, 0, 1, 1, 4096, 128)


def gqa_inputs(ref: Ref):
    hq, hkv, l, d = 4, 2, 4096, 128
    q, k, v = ref.generate_synthetic("mixed", l // 64, 8.0, 7, 1, hq, l, d)
    q = bf16_round(q)
    k = bf16_round(k[:, :hkv])
    v = bf16_round(v[:, :hkv])
    return q, k, v


def expand_kv(x: np.ndarray, hq: int) -> np.ndarray:
    g = hq // x.shape[1]
    return np.repeat(x, g, axis=1)


def make(ref: Ref, q, k, v, cfg: Cfg, path: str) -> None:
    hq = q.shape[1]
    ke, ve = expand_kv(k, hq), expand_kv(v, hq)
    out, tr, plan = ref.attention(q, ke, ve, cfg)
    dense = ref.dense_causal(q, ke, ve)
    l = q.shape[2]
    diff = out.astype(np.float64) - dense.astype(np.float64)
    mse = (diff ** 2).reshape(hq, -1).mean(axis=1)
    mae = np.abs(diff).reshape(hq, -1).mean(axis=1)
    total = l * (l + 1) // 2
    sparsity = 1.0 - (tr.pass1_pairs + tr.pass2_pairs) / total
    np.savez_compressed(
        path,
        q_perm=plan.q_perm.astype(np.int32), kv_perm=plan.kv_perm.astype(np.int32),
        processed=tr.processed.astype(np.int32), pass1_pairs=tr.pass1_pairs,
        pass2_pairs=tr.pass2_pairs, out_rows=out[:, :, ::8, :], out_sha256=np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(out).tobytes()).digest(), np.uint8),
        mse=mse, mae=mae, sparsity=sparsity, cost=np.array(plan.cost, np.int64),
        cfg=np.array([cfg.seg_len, cfg.b_m, cfg.b_n, int(cfg.q_reorder)], np.int64),
        tau=np.array([cfg.tau]))
    print(f"{os.path.basename(path)}: sparsity {sparsity}, mse {mse}, pairs {tr.pass1_pairs} {tr.pass2_pairs}")


def main() -> None:
    build()
    ref = Ref()
    make(ref, *c1_inputs(ref), Cfg(512, 0.005, 64, 64), os.path.join(HERE, "c1_golden.npz"))
    make(ref, *gqa_inputs(ref), Cfg(512, 0.005, 128, 128), os.path.join(HERE, "gqa_golden.npz"))


if __name__ == "__main__":
    main()
