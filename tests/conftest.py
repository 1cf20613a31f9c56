"""Shared pytest fixtures. `-m gpu` tests need a B200; everything else runs on CPU."""
from __future__ import annotations

import json
import os
import sys
from dataclasses import dataclass

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running (large L)")


@dataclass
class Cfg:
    """Duck-typed KernelConfig for the oracle backends."""
    seg_len: int
    tau: float
    b_m: int
    b_n: int
    q_reorder: bool = True
    fused: bool = False
    local_window: int = -1


@pytest.fixture(scope="session")
def oracles():
    from oracle import oracle as orc
    orc.build()
    ref = orc.Ref() if os.path.exists(orc.REF_SO) else None
    return ref, orc.Port()


@pytest.fixture(scope="session")
def port(oracles):
    return oracles[1]


@pytest.fixture(scope="session")
def ref(oracles):
    if oracles[0] is None:
        pytest.skip("reference .so not built (oracle/_ref/libs2o_ref.so)")
    return oracles[0]


@pytest.fixture(scope="session")
def fixtures():
    with open(os.path.join(GOLDEN, "reference_fixtures.json")) as f:
        return json.load(f)


def t4(rows) -> np.ndarray:
    """[[..],..] rows -> fp32 [1,1,L,D]."""
    return np.asarray(rows, np.float32)[None, None]


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_22575_b200 as s2o
    s2o.lib()
    return torch


def assert_trace_ties(backend, q, k, v, cfg, q_perm, kv_perm, got, want, max_frac: float = 0.01):
    """the device trace `got` equals the reference's `want`, except at threshold
    ties -- every differing tile must have the reference's gain at its first differing chunk within
    |gain - tau| / tau <= 1e-4 (oracle.trace_ties). q/k/v are the fp32 arrays the oracle saw (K/V
    expanded to Hq heads), q_perm/kv_perm the (bit-identical) plan. Returns the tie records."""
    from oracle.oracle import trace_ties
    got = np.asarray(got)
    want = np.asarray(want)
    zh = np.asarray(q).shape[0] * np.asarray(q).shape[1]
    n_seg = -(-np.asarray(q).shape[2] // cfg.seg_len)
    ties = trace_ties(backend, q, k, v, cfg, np.asarray(q_perm).reshape(zh, n_seg, -1),
                      np.asarray(kv_perm).reshape(zh, -1), got, want)
    bad = [t for t in ties if not t["tie"]]
    assert not bad, f"trace differences that are not threshold ties: {bad[:5]}"
    assert len(ties) <= max(1, int(max_frac * want.size)), f"too many ties: {len(ties)}"
    return ties
