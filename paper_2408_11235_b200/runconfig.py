"""Scalar conversions of the reference's run configuration (config.cpp:15-52).

Used by ``solver.RunConfig``. Numbers are parsed the way
``std::stod`` / ``std::stoi`` parse them -- libc ``strtod`` / ``strtol`` with
the same range errors -- and must consume the whole value (config.cpp:23-45);
doubles echo as ``%.17g`` (config.cpp:47-51); ``nsteps`` rounds like
``std::lround`` (config.cpp:220).
"""
from __future__ import annotations

import ctypes as C
import math

_libc = C.CDLL(None, use_errno=True)
_libc.strtod.restype = C.c_double
_libc.strtod.argtypes = [C.c_char_p, C.POINTER(C.c_char_p)]
_libc.strtol.restype = C.c_long
_libc.strtol.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_int]
_libc.snprintf.restype = C.c_int

_ERANGE = 34
_INT_MIN, _INT_MAX = -(2 ** 31), 2 ** 31 - 1


def _strto(fn, text: str, *extra):
    raw = text.encode()
    if b"\0" in raw:  # std::string with an embedded NUL: strto* stops there
        raw = raw.split(b"\0", 1)[0] + b"\0"
        full = False
    else:
        full = True
    buf = C.create_string_buffer(raw)
    end = C.c_char_p()
    C.set_errno(0)
    val = fn(buf, C.byref(end), *extra)
    err = C.get_errno()
    used = C.cast(end, C.c_void_p).value - C.addressof(buf)
    return val, err, used, full


def stod_full(key: str, v: str) -> float:
    """to_double (config.cpp:23-33): std::stod + whole-string check."""
    val, err, used, full = _strto(_libc.strtod, v)
    if used == 0 or err == _ERANGE or not full or used != len(v.encode()):
        raise RuntimeError(f"{key}: not a number: '{v}'")
    return val


def stoi_full(key: str, v: str) -> int:
    """to_int (config.cpp:35-45): std::stoi (strtol base 10, int range) + whole-string check."""
    val, err, used, full = _strto(_libc.strtol, v, 10)
    if (used == 0 or err == _ERANGE or not _INT_MIN <= val <= _INT_MAX or not full
            or used != len(v.encode())):
        raise RuntimeError(f"{key}: not an integer: '{v}'")
    return val


def onoff(key: str, v: str) -> bool:
    """to_onoff (config.cpp:47-51)"""
    if v in ("on", "true", "1"):
        return True
    if v in ("off", "false", "0"):
        return False
    raise RuntimeError(f"{key}: expected on|off, got '{v}'")


def g17(v: float) -> str:
    """snprintf("%.17g") (config.cpp:53-57), through libc so nan/-nan/inf print the same."""
    buf = C.create_string_buffer(64)
    _libc.snprintf(buf, 64, b"%.17g", C.c_double(v))
    return buf.value.decode()


def e17(v: float) -> str:
    """snprintf(" % .17e") (tools/solkin_main.cpp:52)"""
    buf = C.create_string_buffer(64)
    _libc.snprintf(buf, 64, b" % .17e", C.c_double(v))
    return buf.value.decode()


def trim(s: str) -> str:
    """config.cpp:15-20 (space, tab, CR, LF)"""
    return s.strip(" \t\r\n")


def lround(x: float) -> int:
    """std::lround: half away from zero (LONG_MIN for nan / inf / overflow, as glibc on x86-64)."""
    if not math.isfinite(x) or abs(x) >= 2.0 ** 63:
        return -(2 ** 63)
    a = abs(x)
    f = math.floor(a)
    r = f + 1 if a - f >= 0.5 else f
    return int(math.copysign(r, x)) if r else 0
