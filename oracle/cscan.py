"""ctypes loader for oracle/scan.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_scan_u8_packed32.argtypes = [_P, _P, _I64, _I64, _I64, _I64, _INT, _INT]
        L.orc_scan_p32.argtypes = [_P, _P, _I64, _I64, _I64, _I64, _INT, _INT]
        L.orc_scan_p32_slab.argtypes = [_P, _P, _P, _P, _I64, _I64, _I64, _INT]
        for f in (L.orc_scan_u8_packed32, L.orc_scan_p32, L.orc_scan_p32_slab):
            f.restype = None
        L.orc_threads.restype = _INT
        _lib = L
    return _lib


def threads() -> int:
    """Worker threads each scan uses (ORACLE_THREADS, default all online cores)."""
    return int(lib().orc_threads())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def scan_u8(images: np.ndarray, fill: int = 1, edgeset: bool = False) -> np.ndarray:
    """uint8 [N, H, W] or [H, W] -> packed uint32 output [N, H, ceil(W/32)] (pad = 1)."""
    a = np.ascontiguousarray(images, dtype=np.uint8)
    squeeze = a.ndim == 2
    if squeeze:
        a = a[None]
    n, h, w = a.shape
    out = np.empty((n, h, -(-w // 32)), dtype=np.uint32)
    lib().orc_scan_u8_packed32(_ptr(a), _ptr(out), n, h, w, w, int(fill), int(edgeset))
    return out[0] if squeeze else out


def scan_p32(words: np.ndarray, width: int, fill: int = 1, edgeset: bool = False) -> np.ndarray:
    """packed uint32 [N, H, S] or [H, S] (S >= ceil(W/32)) -> packed output [.., H, ceil(W/32)]."""
    a = np.ascontiguousarray(words, dtype=np.uint32)
    squeeze = a.ndim == 2
    if squeeze:
        a = a[None]
    n, h, s = a.shape
    out = np.empty((n, h, -(-width // 32)), dtype=np.uint32)
    lib().orc_scan_p32(_ptr(a), _ptr(out), n, h, width, s, int(fill), int(edgeset))
    return out[0] if squeeze else out


def scan_p32_slab(slab: np.ndarray, above, below, width: int, fill: int = 1) -> np.ndarray:
    s = np.ascontiguousarray(slab, dtype=np.uint32)
    rows, stride = s.shape
    ab = None if above is None else np.ascontiguousarray(above, dtype=np.uint32)
    be = None if below is None else np.ascontiguousarray(below, dtype=np.uint32)
    out = np.empty((rows, -(-width // 32)), dtype=np.uint32)
    lib().orc_scan_p32_slab(_ptr(s), None if ab is None else _ptr(ab),
                            None if be is None else _ptr(be), _ptr(out), rows, width, stride,
                            int(fill))
    return out
