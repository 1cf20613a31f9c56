"""The C-ABI boundary without a GPU: the library loads, exports every symbol the header
declares, validates arguments with the reference's messages, and its host-side pieces
(early_stop_check, the synthetic generator, workspace queries) behave like the reference.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, Cfg

import paper_2602_22575_b200 as s2o
from paper_2602_22575_b200 import s2o as api

HEADER = os.path.join(ROOT, "include", "s2o_cuda.h")


def header_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(s2o_[a-z0-9_]+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = s2o.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.s2o_abi_version() == 1


def test_library_is_sm100a_native():
    from paper_2602_22575_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_validation_messages():
    cases = [
        (s2o.KernelConfig(seg_len=0), "segment length must satisfy 1 <= S <= L"),
        (s2o.KernelConfig(seg_len=9), "segment length must satisfy 1 <= S <= L"),
        (s2o.KernelConfig(seg_len=4, tau=-0.1), "tau must be >= 0"),
        (s2o.KernelConfig(seg_len=4, tiles=s2o.TileSpec(0, 2)), "tile sizes must be >= 1"),
        (s2o.KernelConfig(seg_len=4, local_window=5), "local window must satisfy W <= S"),
        (s2o.KernelConfig(seg_len=4, fused=True), "fused variant requires q_reorder = false"),
    ]
    for cfg, msg in cases:
        with pytest.raises(ValueError) as ei:
            cfg.validate(8)
        assert str(ei.value) == msg
    s2o.KernelConfig(seg_len=4, q_reorder=False, fused=True).validate(8)
    with pytest.raises(ValueError):
        s2o.SegmentConfig.for_sequence(4, 5)
    seg = s2o.SegmentConfig.for_sequence(10, 4)
    assert (seg.seg_count, seg.last_len, seg.len(2), seg.prefix_len(2)) == (3, 2, 2, 8)


def test_early_stop_check_host(fixtures):
    f = fixtures["early_stop_check"]
    for tau, want in f["cases"]:
        assert s2o.early_stop_check(f["prev"], f["new"], tau) == want
    with pytest.raises(ValueError, match="uninitialized state"):
        s2o.early_stop_check([0.0, 1.0], f["new"], 0.1)
    with pytest.raises(ValueError, match="normalizer vectors must align"):
        s2o.early_stop_check([], [], 0.1)
    # NaN gains drop out of the max (kernel.cpp:230-231)
    assert s2o.early_stop_check([1.0, 1.0], [float("nan"), 1.0001], 0.01)


@pytest.mark.parametrize("pattern", ["gaussian", "vertical", "horizontal", "slash", "mixed"])
def test_synthetic_bit_identical_to_reference(ref, pattern):
    for (z, h, l, d, stripes, seed) in [(1, 1, 64, 8, 4, 0), (2, 3, 256, 32, 16, 5)]:
        mine = s2o.generate_synthetic(pattern, stripes, 8.0, seed, z, h, l, d, threads=3)
        theirs = ref.generate_synthetic(pattern, stripes, 8.0, seed, z, h, l, d)
        for a, b in zip(mine, theirs):
            np.testing.assert_array_equal(a, b)


def test_synthetic_head_prefix_property():
    """Planted geometry is H-independent, so an H=2 generation equals heads 0..1 of an H=4
    one bit for bit -- this is how GQA K/V are built for the benchmark."""
    a = s2o.generate_synthetic("mixed", 8, 8.0, 1, 1, 4, 128, 16)
    b = s2o.generate_synthetic("mixed", 8, 8.0, 1, 1, 2, 128, 16)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x[:, :2], y)


def _problem(z=1, hq=4, hkv=2, l=1024, d=128, dt=s2o.S2O_BF16):
    p = api._Problem()
    s2o.lib().s2o_problem_init(C.byref(p), C.c_int64(z), C.c_int64(hq), C.c_int64(hkv),
                               C.c_int64(l), C.c_int64(d), C.c_int32(dt), C.c_int32(dt))
    return p


def test_workspace_queries_and_path_selection():
    lib = s2o.lib()
    p = _problem()
    nbytes = C.c_size_t(0)
    assert lib.s2o_plan_workspace_size(C.byref(p), C.c_int64(256), C.byref(nbytes)) == 0
    assert nbytes.value > 0
    cfg = s2o.KernelConfig(seg_len=256)._c()
    assert lib.s2o_attention_workspace_size(C.byref(p), C.byref(cfg), C.byref(nbytes)) == 0
    assert nbytes.value > 4 * 1024 * 128 * 4  # holds the fp32 pass buffers
    out = C.c_int32(0)
    gen = s2o.KernelConfig(seg_len=256, path=s2o.PATH_GENERIC)._c()
    assert lib.s2o_select_path(C.byref(p), C.byref(gen), C.byref(out)) == 0
    assert out.value == s2o.PATH_GENERIC
    # bad GQA ratio and bad segment length are rejected before any device work
    bad = _problem(hq=3, hkv=2)
    assert lib.s2o_plan_workspace_size(C.byref(bad), C.c_int64(256), C.byref(nbytes)) == 9
    assert lib.s2o_plan_workspace_size(C.byref(p), C.c_int64(0), C.byref(nbytes)) == 1
    assert b"segment length" in lib.s2o_last_error()


def test_device_entry_points_reject_bad_args_without_gpu():
    lib = s2o.lib()
    p = _problem()
    cfg = s2o.KernelConfig(seg_len=256, q_reorder=True, fused=True)._c()
    rc = lib.s2o_attention_fwd(C.byref(p), C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), C.byref(cfg),
                               C.c_void_p(1), None, None, None, None, None, None, C.c_size_t(0), None)
    assert rc == 5
    assert lib.s2o_last_error() == b"fused variant requires q_reorder = false"
    cfg = s2o.KernelConfig(seg_len=256)._c()
    rc = lib.s2o_attention_fwd(C.byref(p), C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), C.byref(cfg),
                               C.c_void_p(1), None, None, None, None, None, None, C.c_size_t(16), None)
    assert rc == 16  # workspace too small
