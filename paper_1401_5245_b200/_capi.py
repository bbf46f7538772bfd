"""ctypes binding of `libbitedge_cuda.so` (C ABI declared in include/bitedge.h).

There is deliberately no fallback: if the library is missing, or no CUDA
device is present, every compute entry point raises.  Error codes map to the
reference's exception types: negative codes (invalid arguments) -> ValueError
(bitimage.py:89-97, 188-193 raise ValueError for bad shapes), positive codes
(CUDA errors) -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libbitedge_cuda.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "bitedge.h")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int

BE_LEFT, BE_RIGHT, BE_UP, BE_DOWN = 0, 1, 2, 3
BE_OP_NOT, BE_OP_AND, BE_OP_OR = 0, 1, 2


class be_outputs(ctypes.Structure):
    _fields_ = [("edges", _P), ("edgeset", _P), ("side", _P * 4), ("packed", _P)]


_SIGNATURES = {
    "be_edge_packed_u32": [_P, _P, _I64, _I64, _I64, _I64, _INT, _INT, _P],
    "be_edge_packed_u64": [_P, _P, _I64, _I64, _I64, _I64, _INT, _INT, _P],
    "be_pack_edge_u8": [_P, _P, _I64, _I64, _I64, _I64, _I64, _INT, _P, _P],
    "be_edge_packed_halo_u32": [_P, _P, _P, _P, _I64, _I64, _I64, _INT, _I64, _I64, _P],
    "be_edge_packed_halo_ends_u32": [_P, _P, _P, _P, _I64, _I64, _I64, _INT, _P],
    "be_edges_general": [_P, _INT, _I64, _P, _P, ctypes.POINTER(be_outputs), _INT, _I64, _I64,
                         _I64, _I64, _INT, _I64, _I64, _P],
    "be_pack_u8": [_P, _P, _INT, _I64, _I64, _I64, _I64, _I64, _P],
    "be_unpack_u8": [_P, _P, _INT, _I64, _I64, _I64, _I64, _I64, _P],
    "be_bitop": [_INT, _P, _P, _P, _INT, _I64, _I64, _I64, _I64, _P],
    "be_shift": [_P, _P, _INT, _I64, _I64, _I64, _I64, _INT, _INT, _P],
    "be_shift_and": [_P, _P, _P, _INT, _I64, _I64, _I64, _I64, _INT, _INT, _P],
    "be_count_black": [_P, _P, _INT, _I64, _I64, _I64, _I64, _P],
    "be_scan_edges": [_P, _P, _INT, _I64, _I64, _I64, _I64, _INT, _P],
    "be_threshold_edge_u8": [_P, _P, _I64, _I64, _I64, _I64, _I64, _INT, _INT, _P, _P],
    "be_threshold_u8": [_P, _P, _INT, _I64, _I64, _I64, _I64, _I64, _INT, _P],
    "be_p4_decode": [_P, _P, _INT, _I64, _I64, _I64, _I64, _P],
    "be_p4_encode": [_P, _P, _INT, _I64, _I64, _I64, _I64, _P],
    "be_p4_edges": [_P, _P, _I64, _I64, _I64, _INT, _P, _P],
    "be_ipc_export": [_P, _P, ctypes.POINTER(_I64)],
    "be_ipc_open": [_P, _I64, ctypes.POINTER(_P)],
    "be_ipc_close": [_P, _I64],
    "be_host_edges": [_P, _INT, _P, _I64, _I64, _I64, _INT, ctypes.POINTER(_P),
                      ctypes.POINTER(_P), _I64, _P, _P, _INT],
    "be_host_edges_rows": [_P, _INT, _P, _I64, _I64, _INT, _INT, ctypes.POINTER(_P),
                           ctypes.POINTER(_P), _I64, _P, _P, _INT],
    "be_host_detect_u64": [_P, _I64, _I64, _INT, _INT, _P, _P, _P, _P, _P],
    "be_host_detect_u64_staged": [_P, _I64, _I64, _I64, _INT, _INT, _P, _I64, _P, _I64, _P, _P,
                                  _P],
    "be_reload_knobs": [],
    "be_last_error": [],
    "be_abi_version": [],
    "be_launch_count": [],
}

_lib = None
_lock = threading.Lock()


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(be_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _INT
        lib.be_last_error.restype = ctypes.c_char_p
        lib.be_launch_count.restype = _I64
        if lib.be_abi_version() != 1:
            raise RuntimeError("libbitedge_cuda.so ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().be_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def fn(name: str):
    """The typed foreign function itself (hot callers check the rc only when
    it is nonzero)."""
    return getattr(_lib if _lib is not None else load(), name)


def reload_knobs() -> None:
    """Re-read the BITEDGE_* dispatch knobs (read once per process otherwise)."""
    check(load().be_reload_knobs())


def launch_count() -> int:
    return int(load().be_launch_count())
