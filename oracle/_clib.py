"""ctypes loader for oracle.c (fp64 direct sums).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, fp64, OpenMP).  x86-64-v3 rather than
    -march=native because the built .so travels to the GPU box's host."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared",
                               "-std=c99", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        D = ctypes.POINTER(ctypes.c_double)
        L = ctypes.POINTER(ctypes.c_int64)
        i64, i32 = ctypes.c_int64, ctypes.c_int
        common = [i64, i64, i32, i32, i32, D, D, D]
        _lib.orc_H_window.argtypes = common + [i64, i64, i64, i64, D, D]
        _lib.orc_HT_window.argtypes = common + [i64, i64, i64, i64, D, D]
        _lib.orc_H_points.argtypes = common + [D, i64, L, L, D]
        _lib.orc_HT_points.argtypes = common + [D, i64, L, L, D]
        for f in (_lib.orc_H_window, _lib.orc_HT_window, _lib.orc_H_points, _lib.orc_HT_points):
            f.restype = None
    return _lib


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def lptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
