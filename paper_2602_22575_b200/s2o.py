"""Python mirror of the reference's S2O entry points over the C-ABI (include/s2o_cuda.h).

Same names, argument meaning and error behaviour as proj/include/s2o/{plan,kernel}.hpp:

    build_plan(q, k, seg_len)                 -> (PermutationPlan, RankingCost)   plan.hpp:115-116
    segment_representatives(q, k, seg)        -> Representatives                   plan.hpp:100-102
    pass1_dense_init(q, k, v, cfg)            -> PassBuffers                       kernel.hpp:70-71
    pass2_sparse(q, k, v, bufs, plan, cfg)    -> (out, KernelTrace)                kernel.hpp:83-86
    fused_single_pass(q, k, v, plan, cfg)     -> (out, KernelTrace)                kernel.hpp:92-95
    s2o_attention(q, k, v, cfg)               -> S2oResult                         kernel.hpp:106-107
    early_stop_check(prev, new, tau)          -> bool                              kernel.hpp:77-78
    dense_causal_attention(q, k, v)           -> out (device, S = L)               attention.hpp:42

Tensors are torch CUDA tensors: Q [Z, Hq, L, D], K/V [Z, Hkv, L, D] (GQA when Hkv < Hq),
fp32 or bf16, any (batch, head, token) strides with a unit channel stride. PyTorch only
provides device memory and the current stream; every computation is a kernel of
libs2o_cuda.so. There is no CPU fallback: if the library or a CUDA device is missing the
calls raise.

Exceptions mirror the reference: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::runtime_error -> RuntimeError (message text identical).
"""
from __future__ import annotations

import ctypes as C
import functools
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import build as _build

_LIB: Optional[C.CDLL] = None

S2O_F32, S2O_BF16 = 0, 1
PATH_AUTO, PATH_GENERIC, PATH_TCGEN05 = 0, 1, 2
SCORE_EXACT, SCORE_FAST = 0, 1

_ERR_VALUE = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 14, 15, 16, 19}
_ERR_RUNTIME = {12, 17, 18}


class _Problem(C.Structure):
    _fields_ = [("z", C.c_int64), ("hq", C.c_int64), ("hkv", C.c_int64), ("l", C.c_int64),
                ("d", C.c_int64), ("in_dtype", C.c_int32), ("out_dtype", C.c_int32),
                ("q_stride", C.c_int64 * 3), ("k_stride", C.c_int64 * 3),
                ("v_stride", C.c_int64 * 3), ("o_stride", C.c_int64 * 3)]


class _Config(C.Structure):
    _fields_ = [("seg_len", C.c_int64), ("tau", C.c_double), ("b_m", C.c_int64),
                ("b_n", C.c_int64), ("q_reorder", C.c_int32), ("fused", C.c_int32),
                ("local_window", C.c_int64), ("path", C.c_int32), ("score_mode", C.c_int32),
                ("plan_depth", C.c_int32)]


def lib() -> C.CDLL:
    """Load (building if needed) libs2o_cuda.so. Raises if it cannot be loaded."""
    global _LIB
    if _LIB is None:
        # S2O_LIB_PATH: a prebuilt variant of the library (dev A/B builds); else the in-tree build
        path = os.environ.get("S2O_LIB_PATH") or _build.build()  # no-op when the .so matches its sources
        _LIB = C.CDLL(path)
        _LIB.s2o_last_error.restype = C.c_char_p
        _LIB.s2o_status_string.restype = C.c_char_p
        if _LIB.s2o_abi_version() != 1:
            raise RuntimeError("libs2o_cuda ABI mismatch")
    return _LIB


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().s2o_last_error().decode() or lib().s2o_status_string(rc).decode()
    if rc in _ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


# ----------------------------------------------------------------------------- config
@dataclass
class TileSpec:
    b_m: int = 128
    b_n: int = 128


@dataclass
class KernelConfig:
    """s2o::KernelConfig (kernel.hpp:19-28) plus execution knobs (path, score_mode)."""
    seg_len: int = 128
    tau: float = 0.005
    tiles: TileSpec = field(default_factory=TileSpec)
    q_reorder: bool = True
    fused: bool = False
    local_window: int = -1
    path: int = PATH_AUTO
    score_mode: int = SCORE_EXACT
    plan_depth: int = 0  # s2o_attention: 0 = auto top-6144 kv_perm per segment, -1 = full

    @property
    def b_m(self) -> int:
        return self.tiles.b_m

    @property
    def b_n(self) -> int:
        return self.tiles.b_n

    def _c(self) -> _Config:
        return _Config(int(self.seg_len), float(self.tau), int(self.tiles.b_m), int(self.tiles.b_n),
                       int(bool(self.q_reorder)), int(bool(self.fused)), int(self.local_window),
                       int(self.path), int(self.score_mode), int(self.plan_depth))

    def validate(self, l: int) -> None:
        """KernelConfig::validate (kernel.cpp:166-182)."""
        c = self._c()
        _check(lib().s2o_kernel_config_validate(C.byref(c), C.c_int64(l)))


@dataclass
class SegmentConfig:
    """SegmentConfig (plan.hpp:16-29)."""
    seg_len: int
    seg_count: int
    last_len: int

    @staticmethod
    def for_sequence(l: int, seg_len: int) -> "SegmentConfig":
        if seg_len < 1 or seg_len > l:
            raise ValueError("segment length must satisfy 1 <= S <= L")
        n = (l + seg_len - 1) // seg_len
        return SegmentConfig(seg_len, n, l - (n - 1) * seg_len)

    def begin(self, n: int) -> int:
        return n * self.seg_len

    def len(self, n: int) -> int:
        return self.last_len if n + 1 == self.seg_count else self.seg_len

    def prefix_len(self, n: int) -> int:
        return n * self.seg_len

    @property
    def kv_per_head(self) -> int:
        return self.seg_len * self.seg_count * (self.seg_count - 1) // 2

    def kv_offset(self, n: int) -> int:
        return self.seg_len * n * (n - 1) // 2


@dataclass
class RankingCost:
    dot_products: int = 0
    sort_items: int = 0


@dataclass
class PermutationPlan:
    """Device plan (plan.hpp:81-97): q_perm int32 [Z,Hq,N,S] (segment-local),
    kv_perm int32 [Z,Hq,S*N*(N-1)/2] (absolute ids, segment n at S*n*(n-1)/2)."""
    z: int
    h: int
    seg: SegmentConfig
    q_perm: "torch.Tensor"
    kv_perm: "torch.Tensor"
    guide_source: str = "k_mean[segment 0]"

    def q_perm_at(self, zi: int, hi: int, n: int):
        return self.q_perm[zi, hi, n, : self.seg.len(n)]

    def kv_perm_at(self, zi: int, hi: int, n: int):
        o = self.seg.kv_offset(n)
        return self.kv_perm[zi, hi, o: o + self.seg.prefix_len(n)]


@dataclass
class PassBuffers:
    """Pass-1 state (kernel.hpp:31-47) on the device, fp32: acc [Z,Hq,L,D], ell/m [Z,Hq,L]."""
    acc: "torch.Tensor"
    ell: "torch.Tensor"
    m: "torch.Tensor"


@dataclass
class KernelTrace:
    """KernelTrace (kernel.hpp:52-66): processed int32 [Z,Hq,N,T], pair counters int64 [Z,Hq]."""
    z: int
    h: int
    l: int
    seg_len: int
    tiles: TileSpec
    processed: "torch.Tensor"
    pass1_pairs: "torch.Tensor"
    pass2_pairs: "torch.Tensor"

    def processed_tiles(self) -> list:
        """Nested [z*h][segment][qtile] lists like the reference's processed_tiles."""
        seg = SegmentConfig.for_sequence(self.l, self.seg_len)
        p = self.processed.reshape(self.z * self.h, seg.seg_count, -1).cpu().numpy()
        out = []
        for zh in range(self.z * self.h):
            out.append([[int(x) for x in p[zh, n, : -(-seg.len(n) // self.tiles.b_m)]]
                        for n in range(seg.seg_count)])
        return out


@dataclass
class Representatives:
    q_mean: "torch.Tensor"  # [Z,Hq,N,D] fp32
    k_mean: "torch.Tensor"  # [Z,Hkv,N,D] fp32


@dataclass
class S2oResult:
    out: "torch.Tensor"
    trace: KernelTrace
    plan: PermutationPlan
    cost: RankingCost


# ----------------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return S2O_F32
    if t.dtype == torch.bfloat16:
        return S2O_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


def _check_tensor(t, name: str):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise RuntimeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dim() != 4 or t.stride(3) != 1:
        raise ValueError(f"{name} must be [Z,H,L,D] with a unit channel stride")


def _problem(q, k, v=None, o=None, out_dtype=None) -> _Problem:
    _check_tensor(q, "q")
    _check_tensor(k, "k")
    if v is not None:
        _check_tensor(v, "v")
    z, hq, l, d = q.shape
    hkv = k.shape[1]
    if k.shape[0] != z or k.shape[2] != l or k.shape[3] != d or k.dtype != q.dtype:
        raise ValueError("Q/K/V dims must match")
    if v is not None and (tuple(v.shape) != tuple(k.shape) or v.dtype != q.dtype):
        raise ValueError("Q/K/V dims must match")
    if hq % hkv:
        raise ValueError("Q/K/V dims must match")
    p = _Problem()
    p.z, p.hq, p.hkv, p.l, p.d = z, hq, hkv, l, d
    p.in_dtype = _dtype_code(q)
    p.out_dtype = _dtype_code(o) if o is not None else (out_dtype if out_dtype is not None else S2O_F32)
    for i in range(3):
        p.q_stride[i] = q.stride(i)
        p.k_stride[i] = k.stride(i)
        p.v_stride[i] = (v if v is not None else k).stride(i)
        p.o_stride[i] = (o if o is not None else q).stride(i)
    return p


def _stream(device=None) -> C.c_void_p:
    """The current stream of `device` (the tensors' device, not the current device)."""
    return C.c_void_p(_torch().cuda.current_stream(device).cuda_stream)


def _on(t):
    """Context that makes the tensors' device current for the C-ABI call (the library launches
    on the current device; smem attributes and TMEM are per device)."""
    return _torch().cuda.device(t.device)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


_WS: dict = {}


def _workspace(nbytes: int, device):
    """Cached workspace per (device, current stream), grown on demand. The C-ABI is only safe
    for distinct workspaces across streams, so each stream gets its own; a buffer replaced by
    a larger one is freed through the caching allocator, which orders the free after the work
    already queued on that stream."""
    torch = _torch()
    stream = torch.cuda.current_stream(device)
    key = (device.index if hasattr(device, "index") else device, stream.cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _pass_status(p: _Problem, c: _Config, ws, whole_op: bool) -> None:
    """Device-side errors of the last call ('uninitialized state' kernel.cpp:228, 'uncovered query
    row' kernel.cpp:155): one read of the workspace status word (synchronises the stream)."""
    fn = lib().s2o_attention_status if whole_op else lib().s2o_pass_status
    _check(fn(C.byref(p), C.byref(c), _ptr(ws), C.c_size_t(ws.numel()), _stream()))


def _device_guard(fn):
    """Run a C-ABI wrapper with the device of its first CUDA tensor argument current, so the
    kernels launch on that device and on its current stream."""
    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        t = next((a for a in args if hasattr(a, "is_cuda") and a.is_cuda), None)
        if t is None:
            return fn(*args, **kwargs)
        with _torch().cuda.device(t.device):
            return fn(*args, **kwargs)
    return wrapped


def _out_like(q, out_dtype):
    torch = _torch()
    dt = {S2O_F32: torch.float32, S2O_BF16: torch.bfloat16}[out_dtype]
    return torch.empty(q.shape, dtype=dt, device=q.device)


def _default_out_dtype(q) -> int:
    return _dtype_code(q)


# ----------------------------------------------------------------------------- Step 1
@_device_guard
def segment_representatives(q, k, seg: SegmentConfig) -> Representatives:
    torch = _torch()
    p = _problem(q, k)
    qm = torch.empty((p.z, p.hq, seg.seg_count, p.d), dtype=torch.float32, device=q.device)
    km = torch.empty((p.z, p.hkv, seg.seg_count, p.d), dtype=torch.float32, device=q.device)
    _check(lib().s2o_segment_representatives(C.byref(p), _ptr(q), _ptr(k), C.c_int64(seg.seg_len),
                                             _ptr(qm), _ptr(km), _stream()))
    return Representatives(qm, km)


@_device_guard
def build_plan(q, k, seg_len: int, score_mode: int = SCORE_EXACT):
    """build_plan (plan.cpp:140-162) on the device. Returns (PermutationPlan, RankingCost)."""
    torch = _torch()
    p = _problem(q, k)
    seg = SegmentConfig.for_sequence(p.l, seg_len)
    cfg = KernelConfig(seg_len=seg_len, score_mode=score_mode)._c()
    nbytes = C.c_size_t(0)
    _check(lib().s2o_plan_workspace_size(C.byref(p), C.c_int64(seg_len), C.byref(nbytes)))
    ws = _workspace(nbytes.value, q.device)
    qp = torch.empty((p.z, p.hq, seg.seg_count, seg.seg_len), dtype=torch.int32, device=q.device)
    kv = torch.empty((p.z, p.hq, max(seg.kv_per_head, 1)), dtype=torch.int32, device=q.device)
    cost = (C.c_int64 * 2)()
    _check(lib().s2o_plan_build(C.byref(p), _ptr(q), _ptr(k), C.byref(cfg), _ptr(qp), _ptr(kv),
                                cost, _ptr(ws), C.c_size_t(ws.numel()), _stream()))
    plan = PermutationPlan(p.z, p.hq, seg, qp, kv[:, :, : seg.kv_per_head])
    return plan, RankingCost(int(cost[0]), int(cost[1]))


@_device_guard
def build_plan_truncated(q, k, seg_len: int, depth: int = 6144):
    """Truncated plan (s2o_plan_build_truncated): (q_perm [Z,Hq,N,S], kv_top [Z,Hq,N,depth],
    flag). kv_top[..., n, :min(nS, depth)] == the first entries of the full kv_perm segment."""
    torch = _torch()
    p = _problem(q, k)
    seg = SegmentConfig.for_sequence(p.l, seg_len)
    cfg = KernelConfig(seg_len=seg_len)._c()
    nbytes = C.c_size_t(0)
    _check(lib().s2o_plan_workspace_size(C.byref(p), C.c_int64(seg_len), C.byref(nbytes)))
    ws = _workspace(nbytes.value, q.device)
    qp = torch.empty((p.z, p.hq, seg.seg_count, seg.seg_len), dtype=torch.int32, device=q.device)
    kv = torch.empty((p.z, p.hq, seg.seg_count, depth), dtype=torch.int32, device=q.device)
    flag = torch.zeros(1, dtype=torch.int32, device=q.device)
    _check(lib().s2o_plan_build_truncated(C.byref(p), _ptr(q), _ptr(k), C.byref(cfg), C.c_int64(depth),
                                          _ptr(qp), _ptr(kv), _ptr(flag), _ptr(ws), C.c_size_t(ws.numel()),
                                          _stream()))
    return qp, kv, flag


# ----------------------------------------------------------------------------- Step 2
def _pass_ws(p: _Problem, c: _Config, device):
    nbytes = C.c_size_t(0)
    _check(lib().s2o_pass_workspace_size(C.byref(p), C.byref(c), C.byref(nbytes)))
    return _workspace(nbytes.value, device)


def _trace(p: _Problem, cfg: KernelConfig, device) -> KernelTrace:
    torch = _torch()
    seg = SegmentConfig.for_sequence(p.l, cfg.seg_len)
    t = -(-cfg.seg_len // cfg.tiles.b_m)
    return KernelTrace(p.z, p.hq, p.l, cfg.seg_len, TileSpec(cfg.tiles.b_m, cfg.tiles.b_n),
                       torch.empty((p.z, p.hq, seg.seg_count, t), dtype=torch.int32, device=device),
                       torch.empty((p.z, p.hq), dtype=torch.int64, device=device),
                       torch.empty((p.z, p.hq), dtype=torch.int64, device=device))


@_device_guard
def pass1_dense_init(q, k, v, cfg: KernelConfig) -> PassBuffers:
    torch = _torch()
    p = _problem(q, k, v)
    c = cfg._c()
    _check(lib().s2o_kernel_config_validate(C.byref(c), C.c_int64(p.l)))
    acc = torch.empty((p.z, p.hq, p.l, p.d), dtype=torch.float32, device=q.device)
    ell = torch.empty((p.z, p.hq, p.l), dtype=torch.float32, device=q.device)
    m = torch.empty((p.z, p.hq, p.l), dtype=torch.float32, device=q.device)
    ws = _pass_ws(p, c, q.device)
    _check(lib().s2o_pass1(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.byref(c), _ptr(acc), _ptr(ell),
                           _ptr(m), _ptr(ws), C.c_size_t(ws.numel()), _stream()))
    return PassBuffers(acc, ell, m)


def _check_plan(plan: PermutationPlan, p: _Problem, cfg: KernelConfig) -> None:
    expect = SegmentConfig.for_sequence(p.l, cfg.seg_len)
    if plan.z != p.z or plan.h != p.hq or plan.seg != expect:
        raise ValueError("plan/config mismatch: segment layout differs")


@_device_guard
def pass2_sparse(q, k, v, bufs: PassBuffers, plan: PermutationPlan, cfg: KernelConfig,
                 out=None, check: bool = True):
    o = out if out is not None else _out_like(q, _default_out_dtype(q))
    p = _problem(q, k, v, o)
    c = cfg._c()
    _check(lib().s2o_kernel_config_validate(C.byref(c), C.c_int64(p.l)))
    _check_plan(plan, p, cfg)
    if tuple(bufs.acc.shape) != (p.z, p.hq, p.l, p.d) or tuple(bufs.ell.shape) != (p.z, p.hq, p.l):
        raise ValueError("pass buffers do not match tensor dims")
    tr = _trace(p, cfg, q.device)
    ws = _pass_ws(p, c, q.device)
    kv = plan.kv_perm.contiguous()
    _check(lib().s2o_pass2(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.byref(c), _ptr(bufs.acc),
                           _ptr(bufs.ell), _ptr(bufs.m), _ptr(plan.q_perm.contiguous()),
                           _ptr(kv) if kv.numel() else _ptr(plan.q_perm), _ptr(o), _ptr(tr.processed),
                           _ptr(tr.pass1_pairs), _ptr(tr.pass2_pairs), _ptr(ws),
                           C.c_size_t(ws.numel()), _stream()))
    if check:
        _pass_status(p, c, ws, False)
    return o, tr


@_device_guard
def fused_single_pass(q, k, v, plan: PermutationPlan, cfg: KernelConfig, out=None, check: bool = True):
    if not cfg.fused or cfg.q_reorder:
        raise ValueError("fused variant requires fused = true, q_reorder = false")
    o = out if out is not None else _out_like(q, _default_out_dtype(q))
    p = _problem(q, k, v, o)
    c = cfg._c()
    _check(lib().s2o_kernel_config_validate(C.byref(c), C.c_int64(p.l)))
    _check_plan(plan, p, cfg)
    tr = _trace(p, cfg, q.device)
    ws = _pass_ws(p, c, q.device)
    kv = plan.kv_perm.contiguous()
    _check(lib().s2o_fused(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.byref(c),
                           _ptr(kv) if kv.numel() else _ptr(plan.q_perm), _ptr(o), _ptr(tr.processed),
                           _ptr(tr.pass1_pairs), _ptr(tr.pass2_pairs), _ptr(ws),
                           C.c_size_t(ws.numel()), _stream()))
    if check:
        _pass_status(p, c, ws, False)
    return o, tr


@_device_guard
def attention_workspace_bytes(q, k, v, cfg: KernelConfig) -> int:
    p = _problem(q, k, v)
    c = cfg._c()
    nbytes = C.c_size_t(0)
    _check(lib().s2o_attention_workspace_size(C.byref(p), C.byref(c), C.byref(nbytes)))
    return nbytes.value


@_device_guard
def s2o_attention(q, k, v, cfg: KernelConfig, out=None, want_plan: bool = True, check: bool = True) -> S2oResult:
    """s2o_attention (kernel.cpp:351-369): one C-ABI call (plan + passes) on the current stream of
    q's device. check=True reads the device status word afterwards (one stream synchronisation)
    and raises the reference's exception for an uninitialized state / uncovered row; check=False
    keeps the call fully asynchronous (CUDA-graph capturable)."""
    torch = _torch()
    o = out if out is not None else _out_like(q, _default_out_dtype(q))
    p = _problem(q, k, v, o)
    c = cfg._c()
    _check(lib().s2o_kernel_config_validate(C.byref(c), C.c_int64(p.l)))
    seg = SegmentConfig.for_sequence(p.l, cfg.seg_len)
    tr = _trace(p, cfg, q.device)
    qp = kv = None
    if want_plan:
        qp = torch.empty((p.z, p.hq, seg.seg_count, seg.seg_len), dtype=torch.int32, device=q.device)
        kv = torch.empty((p.z, p.hq, max(seg.kv_per_head, 1)), dtype=torch.int32, device=q.device)
    nbytes = C.c_size_t(0)
    _check(lib().s2o_attention_workspace_size(C.byref(p), C.byref(c), C.byref(nbytes)))
    ws = _workspace(nbytes.value, q.device)
    _check(lib().s2o_attention_fwd(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.byref(c), _ptr(o),
                                   _ptr(qp), _ptr(kv), _ptr(tr.processed), _ptr(tr.pass1_pairs),
                                   _ptr(tr.pass2_pairs), _ptr(ws), C.c_size_t(ws.numel()), _stream()))
    if check:
        _pass_status(p, c, ws, True)
    dots = p.l + seg.kv_per_head
    plan = PermutationPlan(p.z, p.hq, seg, qp, kv[:, :, : seg.kv_per_head] if kv is not None else None)
    return S2oResult(o, tr, plan, RankingCost(dots, dots))


@_device_guard
def dense_causal_attention(q, k, v, out_dtype: int = S2O_F32, path: int = PATH_AUTO):
    """Dense causal attention through the same pass-1 kernels with S = L."""
    torch = _torch()
    o = _out_like(q, out_dtype)
    p = _problem(q, k, v, o)
    cfg = KernelConfig(seg_len=p.l, q_reorder=False, path=path)
    if path == PATH_GENERIC:
        cfg.tiles = TileSpec(64, 64)
    ws = _pass_ws(p, cfg._c(), q.device)
    _check(lib().s2o_dense_causal_fwd(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.c_int32(path),
                                      _ptr(o), _ptr(ws), C.c_size_t(ws.numel()), _stream()))
    return o


@_device_guard
def block_topk_attention(q, k, v, block_rows: int, block_cols: int, topk: int, out=None, path: int = PATH_AUTO):
    """block_topk_attention (baseline.hpp:28-36): the self block plus the `topk` prefix blocks of
    largest causal softmax mass per query block (exact fp64 ranking), masked softmax over them.
    Returns (O, pair_count int64 [Z, Hq]) -- BlockTopkResult."""
    torch = _torch()
    o = out if out is not None else _out_like(q, _default_out_dtype(q))
    p = _problem(q, k, v, o)
    nbytes = C.c_size_t(0)
    _check(lib().s2o_block_topk_workspace_size(C.byref(p), C.c_int64(block_rows), C.c_int64(block_cols),
                                               C.c_int64(topk), C.byref(nbytes)))
    ws = _workspace(nbytes.value, q.device)
    pairs = torch.empty((p.z, p.hq), dtype=torch.int64, device=q.device)
    _check(lib().s2o_block_topk_fwd(C.byref(p), _ptr(q), _ptr(k), _ptr(v), C.c_int64(block_rows),
                                    C.c_int64(block_cols), C.c_int64(topk), C.c_int32(path), _ptr(o), _ptr(pairs),
                                    _ptr(ws), C.c_size_t(ws.numel()), _stream()))
    return o, pairs


@_device_guard
def select_path(q, k, v, cfg: KernelConfig) -> int:
    p = _problem(q, k, v)
    c = cfg._c()
    out = C.c_int32(0)
    _check(lib().s2o_select_path(C.byref(p), C.byref(c), C.byref(out)))
    return out.value


# ----------------------------------------------------------------------------- host-side
def early_stop_check(prev_ell, new_ell, tau: float) -> bool:
    prev = np.ascontiguousarray(prev_ell, dtype=np.float64)
    new = np.ascontiguousarray(new_ell, dtype=np.float64)
    if prev.shape != new.shape or prev.size == 0:
        raise ValueError("normalizer vectors must align")
    stop = C.c_int32(0)
    _check(lib().s2o_early_stop_check(prev.ctypes.data_as(C.c_void_p), new.ctypes.data_as(C.c_void_p),
                                      C.c_int64(prev.size), C.c_double(tau), C.byref(stop)))
    return bool(stop.value)


def generate_synthetic(pattern: str, stripe_count: int, stripe_gain: float, seed: int,
                       z: int, h: int, l: int, d: int, threads: int = 0):
    """generate_synthetic (synthetic.cpp:276-328), bit-identical, multi-threaded host code.
    Returns fp32 numpy arrays (q, k, v) of shape [Z,H,L,D]."""
    q = np.empty((z, h, l, d), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    rc = lib().s2o_synthetic_generate(C.c_char_p(pattern.encode()), C.c_int64(stripe_count),
                                      C.c_double(stripe_gain), C.c_uint64(seed), C.c_int64(z),
                                      C.c_int64(h), C.c_int64(l), C.c_int64(d),
                                      q.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.c_void_p),
                                      v.ctypes.data_as(C.c_void_p), C.c_int32(threads))
    if rc != 0:
        raise ValueError("invalid synthetic spec")
    return q, k, v


def attention_host(q: np.ndarray, k: np.ndarray, v: np.ndarray, cfg: KernelConfig,
                   in_dtype: int = S2O_F32, out: Optional[np.ndarray] = None):
    """s2o_attention on HOST buffers (s2o_attention_host): the reference's calling
    convention. q/k/v are contiguous numpy arrays (fp32, or uint16 bf16 bit patterns with
    in_dtype=S2O_BF16). Returns (out, processed, pass1_pairs, pass2_pairs)."""
    z, hq, l, d = q.shape
    hkv = k.shape[1]
    p = _Problem()
    lib().s2o_problem_init(C.byref(p), C.c_int64(z), C.c_int64(hq), C.c_int64(hkv), C.c_int64(l),
                           C.c_int64(d), C.c_int32(in_dtype), C.c_int32(in_dtype))
    seg = SegmentConfig.for_sequence(l, cfg.seg_len)
    t = -(-cfg.seg_len // cfg.tiles.b_m)
    if out is None:
        out = np.empty(q.shape, np.float32 if in_dtype == S2O_F32 else np.uint16)
    proc = np.empty((z, hq, seg.seg_count, t), np.int32)
    p1 = np.empty((z, hq), np.int64)
    p2 = np.empty((z, hq), np.int64)
    c = cfg._c()
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    _check(lib().s2o_attention_host(C.byref(p), vp(q), vp(k), vp(v), C.byref(c), vp(out), None, None,
                                    vp(proc), vp(p1), vp(p2)))
    return out, proc, p1, p2


def attention_host_ptr(q_host, k_host, v_host, o_host, cfg: KernelConfig) -> None:
    """s2o_attention_host on torch CPU tensors (pinned or pageable, fp32 or bf16, dense
    [Z,H,L,D]): host->device copies, the whole operator and the device->host copy of O in
    one C-ABI call. Raises on any error."""
    torch = _torch()
    z, hq, l, d = q_host.shape
    hkv = k_host.shape[1]
    dt = _dtype_code(q_host)
    p = _Problem()
    lib().s2o_problem_init(C.byref(p), C.c_int64(z), C.c_int64(hq), C.c_int64(hkv), C.c_int64(l),
                           C.c_int64(d), C.c_int32(dt), C.c_int32(_dtype_code(o_host)))
    c = cfg._c()
    _check(lib().s2o_attention_host(C.byref(p), _ptr(q_host), _ptr(k_host), _ptr(v_host), C.byref(c),
                                    _ptr(o_host), None, None, None, None, None))
