"""Loader for the sm_100a C-ABI library.

The ctypes signatures are derived from include/stencilgrad_b200.h itself, so
the Python side cannot drift from the C boundary.  There is no fallback: if
the shared object is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
HEADER = os.path.join(ROOT, "include", "stencilgrad_b200.h")
LIB_PATH = os.environ.get("SGB_LIB_PATH") or os.path.join(PKG, "libstencilgrad_b200.so")

SGB_GUARD = 1
SGB_EINVAL = -10000

_CTYPES = {
    "int": ctypes.c_int,
    "double": ctypes.c_double,
    "long long": ctypes.c_longlong,
    "uint64_t": ctypes.c_uint64,
    "unsigned long long": ctypes.c_ulonglong,
    "sgb_stream_t": ctypes.c_void_p,
    "float*": ctypes.c_void_p,
    "double*": ctypes.c_void_p,
    "const double*": ctypes.c_void_p,
    "const float*": ctypes.c_void_p,
    "void**": ctypes.c_void_p,
    "void*": ctypes.c_void_p,
    "const void*": ctypes.c_void_p,
    "long long*": ctypes.c_void_p,
    "int*": ctypes.c_void_p,
    "const char*": ctypes.c_char_p,
    "sgb_plan*": ctypes.c_void_p,
    "sgb_slab*": ctypes.c_void_p,
    "const sgb_slab*": ctypes.c_void_p,
    "sgb_jit_kernel*": ctypes.c_void_p,
    "sgb_jit_kernel**": ctypes.c_void_p,
    "unsigned": ctypes.c_uint,
    "void": None,
}

_PROTO = re.compile(r"^(?P<ret>[A-Za-z_][\w ]*?\**)\s+(?P<name>\w+)\((?P<args>[^;]*?)\);",
                    re.M | re.S)


def parse_header(path: str = HEADER):
    """Returns {name: (ret_type, [(type, param_name), ...])} for every prototype."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    out = {}
    for m in _PROTO.finditer(text):
        ret = " ".join(m.group("ret").split())
        if ret.startswith("typedef") or ret.startswith("#"):
            continue
        args = " ".join(m.group("args").split())
        params = []
        if args and args != "void":
            for a in args.split(","):
                a = a.strip()
                mm = re.match(r"(.*?)(\w+)$", a)
                typ = mm.group(1).replace(" *", "*").strip()
                typ = re.sub(r"\s*\*", "*", typ)
                params.append((typ, mm.group(2)))
        out[m.group("name")] = (ret.replace(" *", "*"), params)
    return out


PROTOTYPES = parse_header()


class LibraryMissing(RuntimeError):
    pass


class StencilError(RuntimeError):
    pass


class GuardViolation(StencilError):
    """The reference's minimum-extent guard failed (emitted code returns 1)."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_1907_02818_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (ret, params) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = _CTYPES[ret]
            fn.argtypes = [_CTYPES[t] for t, _ in params]
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc == SGB_GUARD:
        raise GuardViolation(f"{what}: minimum extent violated (reference guard)")
    msg = lib().sgb_last_error().decode(errors="replace")
    raise StencilError(f"{what} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(lib().sgb_launch_count())
