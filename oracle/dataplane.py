"""ORACLE (test infrastructure): ctypes binding of oracle/dataplane.c."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = C.CDLL(LIB)
        h.lp_ref_fill.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int]
        h.lp_ref_fill.restype = None
        h.lp_ref_checksum.argtypes = [C.c_void_p, C.c_int64]
        h.lp_ref_checksum.restype = C.c_uint64
        h.lp_ref_execute.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int64,
                                     C.POINTER(C.c_uint8), C.c_int]
        h.lp_ref_execute.restype = C.c_int64
        _lib = h
    return _lib


def fill_tensor(numel: int, tensor_id: int, seed: int, kind: int, scale_exp: int) -> np.ndarray:
    """bf16 bits (uint16) of one synthetic tensor."""
    out = np.empty(numel, dtype=np.uint16)
    lib().lp_ref_fill(out.ctypes.data, numel, tensor_id, seed, kind, scale_exp)
    return out


def fill_image(layout, seed: int) -> np.ndarray:
    """The whole packed weight image as bytes (uint8), built on the CPU."""
    img = np.zeros(layout.weights_bytes, dtype=np.uint8)
    for t in layout.tensors:
        bits = fill_tensor(t.numel, t.index, seed, t.kind, t.scale_exp)
        img[t.offset:t.offset + t.nbytes] = bits.view(np.uint8)
    return img


def checksum(buf: np.ndarray) -> int:
    buf = np.ascontiguousarray(buf)
    return int(lib().lp_ref_checksum(buf.ctypes.data, buf.nbytes))


def block_checksums(img: np.ndarray, offsets, lengths) -> list:
    return [checksum(img[o:o + n]) for o, n in zip(offsets, lengths)]


def execute(images: list, offsets, lengths, lines: list, sources: list, threads: int = 0) -> None:
    """Run schedule lines on host images in place; raise on a causality breach."""
    n_nodes, n_blocks = len(images), len(offsets)
    rows = sorted(tuple(int(x) for x in ln.split(",")) for ln in lines)
    flat = (C.c_int32 * (4 * len(rows)))(*[v for r in rows for v in r])
    holds = np.zeros(n_nodes * n_blocks, dtype=np.uint8)
    for s in sources:
        holds[s * n_blocks:(s + 1) * n_blocks] = 1
    ptrs = (C.c_void_p * n_nodes)(*[im.ctypes.data for im in images])
    off = (C.c_int64 * n_blocks)(*offsets)
    ln = (C.c_int64 * n_blocks)(*lengths)
    rc = lib().lp_ref_execute(n_nodes, ptrs, n_blocks, off, ln, flat, len(rows),
                              holds.ctypes.data_as(C.POINTER(C.c_uint8)), threads)
    if rc < 0:
        raise RuntimeError(f"oracle: transfer {-rc - 1} violates causality or bounds: {rows[-rc - 1]}")
