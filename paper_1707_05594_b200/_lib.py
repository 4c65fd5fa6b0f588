"""ctypes loader for libtuckerplan_b200.so (the C ABI in include/tuckerplan_b200.h).

There is no fallback: if the shared library is missing the import fails loudly,
and device entry points return TP_ERR_CUDA when no B200 is present.
"""
from __future__ import annotations

import ctypes
import enum
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libtuckerplan_b200.so")

u64 = ctypes.c_uint64
u64_p = ctypes.POINTER(u64)
int_p = ctypes.POINTER(ctypes.c_int)
size_p = ctypes.POINTER(ctypes.c_size_t)
dbl_p = ctypes.POINTER(ctypes.c_double)
dbl_pp = ctypes.POINTER(dbl_p)


class Errc(enum.IntEnum):
    """tuckerplan::Errc (reference errors.hpp:16-30); value = C status code = ordinal + 1."""
    bad_dims = 1
    k_too_large = 2
    overflow = 3
    bad_tree = 4
    bad_mode = 5
    shape_mismatch = 6
    invalid_grid = 7
    no_valid_grid = 8
    missing_assignment = 9
    too_large = 10
    zero_tensor = 11
    needs_chain_tree = 12
    bad_argument = 13
    cuda = 100
    nccl = 101
    capacity = 102
    internal = 103


class TuckerplanError(RuntimeError):
    """tuckerplan::Error (reference errors.hpp:32-43)."""

    def __init__(self, status: int, what: str, mode: int = -1):
        super().__init__(what)
        try:
            self.code = Errc(status)
        except ValueError:
            self.code = Errc.internal
        self.status = status
        self.mode = mode


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1707_05594_b200/csrc` (there is no CPU fallback)")
    return ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)


lib = _load()
lib.tp_last_error.restype = ctypes.c_char_p
lib.tp_version.restype = ctypes.c_char_p
lib.tp_last_error_mode.restype = ctypes.c_int


def check(status: int) -> None:
    if status != 0:
        raise TuckerplanError(status, lib.tp_last_error().decode("utf-8", "replace"), lib.tp_last_error_mode())


def u64_array(values):
    values = [int(v) for v in values]
    return (u64 * len(values))(*values)


def int_array(values):
    values = [int(v) for v in values]
    return (ctypes.c_int * len(values))(*values)


def size_array(values):
    values = [int(v) for v in values]
    return (ctypes.c_size_t * len(values))(*values)


def exported_symbols_from_header():
    """Names of every `int tp_*(`/`const char* tp_*(`/`void* tp_*(` declared in include/tuckerplan_b200.h."""
    import re
    header = os.path.join(os.path.dirname(_HERE), "include", "tuckerplan_b200.h")
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)))
