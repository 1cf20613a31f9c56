"""S2OT tensor files -- the reference's input/output carrier (tensor_io.cpp:32-83).

Layout (little-endian): b"S2OT", u32 version = 1, u32 Z, H, L, D, then Z*H*L*D fp32 values in
[Z, H, L, D] row-major order. Errors carry the reference's messages (RuntimeError for its
std::runtime_error). Host-side numpy only: the files feed the device path through the usual
host -> device copy.
"""
from __future__ import annotations

import os
import struct

import numpy as np

_MAGIC = b"S2OT"
_VERSION = 1
_HEADER = struct.Struct("<4s5I")  # magic, version, z, h, l, d


def save_tensor_file(t, path) -> None:
    """save_tensor_file (tensor_io.cpp:32-49): a [Z,H,L,D] array (any float dtype) as fp32."""
    a = np.ascontiguousarray(np.asarray(t, dtype=np.float32))
    if a.ndim != 4:
        raise ValueError("an S2OT tensor is 4-D [Z, H, L, D]")
    path = os.fspath(path)
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError("cannot open for writing: " + path) from None
    try:
        with f:
            f.write(_HEADER.pack(_MAGIC, _VERSION, *(int(x) for x in a.shape)))
            f.write(a.astype("<f4", copy=False).tobytes())
    except OSError:
        raise RuntimeError("write failed: " + path) from None


def load_tensor_file(path) -> np.ndarray:
    """load_tensor_file (tensor_io.cpp:51-81): fp32 [Z,H,L,D]; the whole file must be the tensor."""
    path = os.fspath(path)
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError:
        raise RuntimeError("cannot open: " + path) from None
    if len(blob) < 4 or blob[:4] != _MAGIC:
        raise RuntimeError("not an S2OT file")
    if len(blob) < 8 or struct.unpack_from("<I", blob, 4)[0] != _VERSION:
        raise RuntimeError("unsupported version")
    if len(blob) < _HEADER.size:
        raise RuntimeError("size mismatch")
    _, _, z, h, l, d = _HEADER.unpack_from(blob, 0)
    if min(z, h, l, d) < 1:
        raise RuntimeError("size mismatch")
    n = z * h * l * d
    if len(blob) != _HEADER.size + 4 * n:  # short data or trailing bytes
        raise RuntimeError("size mismatch")
    return np.frombuffer(blob, dtype="<f4", count=n, offset=_HEADER.size).astype(np.float32).reshape(z, h, l, d)


def load_trio(base) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """<base>.{q,k,v}.s2ot as the sweep loads them (sweep.cpp:38-45)."""
    q = load_tensor_file(f"{base}.q.s2ot")
    k = load_tensor_file(f"{base}.k.s2ot")
    v = load_tensor_file(f"{base}.v.s2ot")
    if not (q.shape == k.shape == v.shape):
        raise RuntimeError("input tensor trio has mismatched dims")
    return q, k, v
