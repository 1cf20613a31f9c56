"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes/numpy front end for the two CPU checkers built by oracle/Makefile:

* ``Ref``  -> oracle/_ref/libs2o_ref.so: the unmodified reference sources
  (/root/reference/proj/src) behind oracle/ref_capi.cpp.
* ``Port`` -> oracle/_ref/libs2o_oracle.so: the plain-C fp64 restatement
  (oracle/s2o_oracle.c), pinned against Ref and the reference's golden vectors
  by tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  Both backends expose the same numpy-level API
(fp32 [Z,H,L,D] tensors, int64 plans/traces, fp64 pass buffers) -- see the
layout comment at the top of oracle/ref_capi.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libs2o_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libs2o_oracle.so")

_i64 = C.c_int64
_f64 = C.c_double
_ptr = C.c_void_p


def build(force: bool = False) -> None:
    """Compile the checkers (reference .so only when /root/reference exists)."""
    targets = ["restatement"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    if force or not all(os.path.exists(p) for p in (PORT_SO,) + ((REF_SO,) if "ref" in targets else ())):
        subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_ptr)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.msg = msg


@dataclass
class SegCfg:
    seg_len: int
    seg_count: int
    last_len: int

    @staticmethod
    def of(l: int, s: int) -> "SegCfg":
        n = (l + s - 1) // s
        return SegCfg(s, n, l - (n - 1) * s)

    def len(self, n: int) -> int:
        return self.last_len if n + 1 == self.seg_count else self.seg_len

    @property
    def kv_per_head(self) -> int:
        return self.seg_len * self.seg_count * (self.seg_count - 1) // 2

    def kv_offset(self, n: int) -> int:
        return self.seg_len * n * (n - 1) // 2


@dataclass
class Plan:
    q_perm: np.ndarray   # int64 [ZH, N, S]
    kv_perm: np.ndarray  # int64 [ZH, S*N*(N-1)/2]
    cost: tuple[int, int] | None = None


@dataclass
class Trace:
    processed: np.ndarray    # int64 [ZH, N, T]
    pass1_pairs: np.ndarray  # int64 [ZH]
    pass2_pairs: np.ndarray  # int64 [ZH]


class _Backend:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _call(self, name: str, *args):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = C.c_int
        rc = fn(*args)
        if rc != 0:
            raise OracleError(rc, getattr(self.lib, self.prefix + "last_error")().decode())

    @staticmethod
    def _t(x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        assert x.ndim == 4
        return x

    # -- plan ---------------------------------------------------------------
    def argsort_desc_stable(self, scores) -> np.ndarray:
        s = np.ascontiguousarray(scores, dtype=np.float64)
        out = np.empty(max(len(s), 1), np.int64)
        self._call("argsort_desc_stable", _p(s), _i64(len(s)), _p(out))
        return out[: len(s)]

    def early_stop_check(self, prev, new, tau: float) -> bool:
        p = np.ascontiguousarray(prev, dtype=np.float64)
        n = np.ascontiguousarray(new, dtype=np.float64)
        stop = C.c_int(0)
        self._call("early_stop_check", _p(p), _p(n), _i64(len(p)), _f64(tau), C.byref(stop))
        return bool(stop.value)

    def segment_representatives(self, q, k, seg_len: int):
        q, k = self._t(q), self._t(k)
        z, h, l, d = q.shape
        seg = SegCfg.of(l, seg_len) if 1 <= seg_len <= l else SegCfg(seg_len, 1, 1)
        qm = np.zeros((z, h, seg.seg_count, d), np.float32)
        km = np.zeros_like(qm)
        self._call("segment_representatives", _p(q), _p(k), _i64(z), _i64(h), _i64(l), _i64(d),
                   _i64(seg_len), _p(qm), _p(km))
        return qm, km

    def build_plan(self, q, k, seg_len: int) -> Plan:
        q, k = self._t(q), self._t(k)
        z, h, l, d = q.shape
        seg = SegCfg.of(l, seg_len) if 1 <= seg_len <= l else SegCfg(max(seg_len, 1), 1, 1)
        qp = np.zeros((z * h, seg.seg_count, seg.seg_len), np.int64)
        kv = np.zeros((z * h, max(seg.kv_per_head, 1)), np.int64)
        cost = np.zeros(2, np.int64)
        self._call("build_plan", _p(q), _p(k), _i64(z), _i64(h), _i64(l), _i64(d), _i64(seg_len),
                   _p(qp), _p(kv), _p(cost))
        return Plan(qp, kv[:, : seg.kv_per_head].copy(), (int(cost[0]), int(cost[1])))

    # -- kernel -------------------------------------------------------------
    @staticmethod
    def _cfg_args(cfg):
        return (_i64(cfg.seg_len), _f64(cfg.tau), _i64(cfg.b_m), _i64(cfg.b_n),
                C.c_int(int(cfg.q_reorder)), C.c_int(int(cfg.fused)), _i64(cfg.local_window))

    def pass1(self, q, k, v, cfg):
        q, k, v = self._t(q), self._t(k), self._t(v)
        z, h, l, d = q.shape
        acc = np.zeros((z, h, l, d), np.float64)
        ell = np.zeros((z, h, l), np.float64)
        m = np.zeros((z, h, l), np.float64)
        self._call("pass1", _p(q), _p(k), _p(v), _i64(z), _i64(h), _i64(l), _i64(d),
                   *self._cfg_args(cfg), _p(acc), _p(ell), _p(m))
        return acc, ell, m

    def _trace_bufs(self, z, h, l, cfg):
        seg = SegCfg.of(l, cfg.seg_len)
        t = (cfg.seg_len + cfg.b_m - 1) // cfg.b_m
        return Trace(np.zeros((z * h, seg.seg_count, t), np.int64), np.zeros(z * h, np.int64),
                     np.zeros(z * h, np.int64))

    def pass2(self, q, k, v, bufs, plan: Plan, cfg):
        q, k, v = self._t(q), self._t(k), self._t(v)
        z, h, l, d = q.shape
        acc, ell, m = (np.ascontiguousarray(b, dtype=np.float64) for b in bufs)
        out = np.zeros((z, h, l, d), np.float32)
        tr = self._trace_bufs(z, h, l, cfg)
        kv = np.ascontiguousarray(plan.kv_perm, np.int64)
        if kv.size == 0:
            kv = np.zeros(1, np.int64)
        self._call("pass2", _p(q), _p(k), _p(v), _i64(z), _i64(h), _i64(l), _i64(d),
                   *self._cfg_args(cfg), _p(acc), _p(ell), _p(m),
                   _p(np.ascontiguousarray(plan.q_perm, np.int64)), _p(kv), _p(out),
                   _p(tr.processed), _p(tr.pass1_pairs), _p(tr.pass2_pairs))
        return out, tr

    def fused(self, q, k, v, plan: Plan, cfg):
        q, k, v = self._t(q), self._t(k), self._t(v)
        z, h, l, d = q.shape
        out = np.zeros((z, h, l, d), np.float32)
        tr = self._trace_bufs(z, h, l, cfg)
        kv = np.ascontiguousarray(plan.kv_perm, np.int64)
        if kv.size == 0:
            kv = np.zeros(1, np.int64)
        self._call("fused", _p(q), _p(k), _p(v), _i64(z), _i64(h), _i64(l), _i64(d),
                   *self._cfg_args(cfg), _p(np.ascontiguousarray(plan.q_perm, np.int64)), _p(kv),
                   _p(out), _p(tr.processed), _p(tr.pass1_pairs), _p(tr.pass2_pairs))
        return out, tr

    def attention(self, q, k, v, cfg):
        q, k, v = self._t(q), self._t(k), self._t(v)
        z, h, l, d = q.shape
        seg = SegCfg.of(l, cfg.seg_len) if 1 <= cfg.seg_len <= l else SegCfg(max(cfg.seg_len, 1), 1, 1)
        out = np.zeros((z, h, l, d), np.float32)
        qp = np.zeros((z * h, seg.seg_count, seg.seg_len), np.int64)
        kv = np.zeros((z * h, max(seg.kv_per_head, 1)), np.int64)
        cost = np.zeros(2, np.int64)
        tr = self._trace_bufs(z, h, l, cfg) if 1 <= cfg.seg_len <= l and cfg.b_m >= 1 else \
            Trace(np.zeros(1, np.int64), np.zeros(z * h, np.int64), np.zeros(z * h, np.int64))
        self._call("attention", _p(q), _p(k), _p(v), _i64(z), _i64(h), _i64(l), _i64(d),
                   *self._cfg_args(cfg), _p(out), _p(qp), _p(kv), _p(tr.processed),
                   _p(tr.pass1_pairs), _p(tr.pass2_pairs), _p(cost))
        plan = Plan(qp, kv[:, : seg.kv_per_head].copy(), (int(cost[0]), int(cost[1])))
        return out, tr, plan


    def tile_gains(self, qh, kh, vh, seg_len: int, b_n: int, rows, n: int, kv_seg, nchunks: int) -> np.ndarray:
        """Max relative normaliser gain of each of the first `nchunks` kv_perm chunks of one query
        tile, every chunk committed (SURVEY.md §8c P2 evidence). qh/kh/vh: one head [L, D];
        rows: the tile's segment-local query rows; kv_seg: kv_perm[n] (absolute token ids)."""
        qh = np.ascontiguousarray(qh, np.float32)
        kh = np.ascontiguousarray(kh, np.float32)
        vh = np.ascontiguousarray(vh, np.float32)
        rows = np.ascontiguousarray(rows, np.int64)
        kv = np.ascontiguousarray(kv_seg, np.int64)
        if kv.size == 0:
            kv = np.zeros(1, np.int64)
        out = np.zeros(max(nchunks, 1), np.float64)
        self._call("tile_gains", _p(qh), _p(kh), _p(vh), _i64(qh.shape[0]), _i64(qh.shape[1]), _i64(seg_len),
                   _i64(b_n), _p(rows), _i64(len(rows)), _i64(n), _p(kv), _i64(nchunks), _p(out))
        return out[:nchunks]


class Ref(_Backend):
    """The compiled reference (oracle/_ref/libs2o_ref.so)."""
    prefix = "ref_"

    def __init__(self):
        super().__init__(REF_SO)

    def dense_causal(self, q, k, v):
        q, k, v = self._t(q), self._t(k), self._t(v)
        out = np.zeros_like(q)
        self._call("dense_causal", _p(q), _p(k), _p(v), *(_i64(x) for x in q.shape), _p(out))
        return out

    def generate_synthetic(self, pattern: str, stripe_count: int, gain: float, seed: int,
                           z: int, h: int, l: int, d: int):
        q = np.zeros((z, h, l, d), np.float32)
        k = np.zeros_like(q)
        v = np.zeros_like(q)
        self._call("generate_synthetic", C.c_char_p(pattern.encode()), _i64(stripe_count),
                   _f64(gain), C.c_uint64(seed), _i64(z), _i64(h), _i64(l), _i64(d), _p(q), _p(k), _p(v))
        return q, k, v

    def save_tensor(self, path: str, x: np.ndarray) -> None:
        x = self._t(x)
        self._call("save_tensor", C.c_char_p(str(path).encode()), _p(x), *(_i64(v) for v in x.shape))

    def load_tensor(self, path: str) -> np.ndarray:
        dims = np.zeros(4, np.int64)
        self._call("load_tensor", C.c_char_p(str(path).encode()), _p(dims), None)
        out = np.zeros(tuple(int(v) for v in dims), np.float32)
        self._call("load_tensor", C.c_char_p(str(path).encode()), _p(dims), _p(out))
        return out

    def block_topk(self, q, k, v, block_rows: int, block_cols: int, topk: int):
        """block_topk_attention (baseline.cpp): (out fp32 [Z,H,L,D], computed pairs int64 [Z*H])."""
        q, k, v = self._t(q), self._t(k), self._t(v)
        out = np.zeros_like(q)
        pairs = np.zeros(q.shape[0] * q.shape[1], np.int64)
        self._call("block_topk", _p(q), _p(k), _p(v), *(_i64(x) for x in q.shape), _i64(block_rows),
                   _i64(block_cols), _i64(topk), _p(out), _p(pairs))
        return out, pairs

    def run_sweep(self, pattern: str, stripe_count: int, gain: float, seed: int, dims, variants, seg_lens, taus,
                  tiles, topk, block, dump_plan: bool, out_base: str) -> None:
        """run_sweep (sweep.cpp) on a synthetic input: writes <out_base>.{json,csv}."""
        seg = np.asarray(seg_lens, np.int64)
        tau = np.asarray(taus, np.float64)
        tk = np.asarray(topk if topk else [0], np.int64)
        self._call("run_sweep", C.c_char_p(pattern.encode()), _i64(stripe_count), _f64(gain), C.c_uint64(seed),
                   *(_i64(x) for x in dims), C.c_char_p(",".join(variants).encode()), _p(seg), _i64(len(seg)),
                   _p(tau), _i64(len(tau)), _i64(tiles[0]), _i64(tiles[1]), _p(tk), _i64(len(topk)),
                   _i64(block[0]), _i64(block[1]), C.c_int(1 if dump_plan else 0), C.c_char_p(out_base.encode()))

    def rng_normals(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._call("rng_normals", C.c_uint64(seed), _i64(n), _p(out))
        return out

    def mix_seed(self, seed: int, a: int, b: int = 0, c: int = 0) -> int:
        fn = self.lib.ref_mix_seed
        fn.restype = C.c_uint64
        fn.argtypes = [C.c_uint64] * 4
        return int(fn(seed, a, b, c))


class Port(_Backend):
    """The plain-C restatement (oracle/_ref/libs2o_oracle.so)."""
    prefix = "orc_"

    def __init__(self):
        super().__init__(PORT_SO)

    def dense_causal_rows(self, q, k, v, row_begin: int, row_end: int):
        q, k, v = self._t(q), self._t(k), self._t(v)
        z, h, l, d = q.shape
        out = np.zeros((z, h, row_end - row_begin, d), np.float32)
        self._call("dense_causal_rows", _p(q), _p(k), _p(v), _i64(z), _i64(h), _i64(l), _i64(d),
                   _i64(row_begin), _i64(row_end), _p(out))
        return out

    def dense_causal(self, q, k, v):
        return self.dense_causal_rows(q, k, v, 0, np.asarray(q).shape[2])

    def masked_softmax_row(self, q_row, k_head, v_head, visible) -> np.ndarray:
        qr = np.ascontiguousarray(q_row, np.float32)
        kh = np.ascontiguousarray(k_head, np.float32)
        vh = np.ascontiguousarray(v_head, np.float32)
        vis = np.ascontiguousarray(visible, np.int64)
        out = np.zeros(qr.shape[-1], np.float64)
        self._call("masked_softmax_row", _p(qr), _p(kh), _p(vh), _i64(qr.shape[-1]), _p(vis),
                   _i64(len(vis)), _p(out))
        return out


def visible_sets(plan: Plan, trace: Trace, cfg, l: int, zh: int) -> list[list[int]]:
    """Per-row visible key sets from plan + trace (proj/tests/oracles.hpp:84-115)."""
    seg = SegCfg.of(l, cfg.seg_len)
    sets: list[list[int]] = [[] for _ in range(l)]
    for n in range(seg.seg_count):
        begin, ln = n * seg.seg_len, seg.len(n)
        qp = plan.q_perm[zh, n, :ln] if cfg.q_reorder else np.arange(ln)
        kv = plan.kv_perm[zh, seg.kv_offset(n): seg.kv_offset(n) + n * seg.seg_len]
        for tile, t0 in enumerate(range(0, ln, cfg.b_m)):
            tn = min(cfg.b_m, ln - t0)
            committed = int(trace.processed[zh, n, tile])
            take = min(committed * cfg.b_n, len(kv))
            for r in range(tn):
                row = begin + int(qp[t0 + r])
                vis = list(range(begin, row + 1)) + [int(x) for x in kv[:take]]
                sets[row] = sorted(vis)
    return sets


TIE_RTOL = 1e-4  # a trace difference must sit at a threshold tie |gain - tau| / tau <= 1e-4


def trace_ties(backend: _Backend, q, k, v, cfg, q_perm, kv_perm, got, want, zh_list=None) -> list[dict]:
    """Explain every (head, segment, tile) whose committed chunk count differs between `got` (the
    device trace) and `want` (the reference's): replay the tile in the reference arithmetic
    (Backend.tile_gains), take the gain of the first chunk the two decided differently
    (k = min(got, want); both committed chunks 0..k-1), and report it with its distance to tau.

    q/k/v: fp32 [Z, H, L, D] as the reference saw them (K/V already expanded to H heads);
    q_perm int [ZH, N, S] / kv_perm int [ZH, S*N*(N-1)/2] (the reference's plan, identical to the
    device plan); got/want int [ZH, N, T]. Returns one dict per differing tile with 'tie' = whether
    |gain - tau| / tau <= TIE_RTOL."""
    q = np.asarray(q)
    z, h, l, d = q.shape
    seg = SegCfg.of(l, cfg.seg_len)
    got = np.asarray(got).reshape(z * h, seg.seg_count, -1)
    want = np.asarray(want).reshape(z * h, seg.seg_count, -1)
    out = []
    for zh, n, t in zip(*np.nonzero(got != want)):
        if zh_list is not None and zh not in zh_list:
            continue
        zi, hi = divmod(int(zh), h)
        ln = seg.len(int(n))
        t0 = int(t) * cfg.b_m
        tn = min(cfg.b_m, ln - t0)
        rows = (np.asarray(q_perm)[zh, n, t0:t0 + tn] if cfg.q_reorder else np.arange(t0, t0 + tn))
        off = seg.kv_offset(int(n))
        kv = np.asarray(kv_perm)[zh, off: off + int(n) * seg.seg_len]
        kc = int(min(got[zh, n, t], want[zh, n, t]))
        gains = backend.tile_gains(q[zi, hi], np.asarray(k)[zi, hi], np.asarray(v)[zi, hi], cfg.seg_len, cfg.b_n,
                                   rows, int(n), kv, kc + 1)
        g = float(gains[kc])
        rel = abs(g - cfg.tau) / cfg.tau if cfg.tau > 0 else float("inf")
        out.append({"zh": int(zh), "segment": int(n), "tile": int(t), "got": int(got[zh, n, t]),
                    "want": int(want[zh, n, t]), "gain": g, "rel_to_tau": rel, "tie": bool(rel <= TIE_RTOL)})
    return out
