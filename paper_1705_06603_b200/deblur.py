"""Thin ctypes binding of libdeblur (include/deblur.h): argument marshalling only.

Every step of the hot path runs in libdeblur's CUDA kernels.  There is no CPU
or PyTorch fallback: if the library cannot be loaded this module raises, and
deblur_create fails with DEBLUR_ECUDA on a machine without an sm_100 GPU.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdeblur.so")

ABI_VERSION = 3
OP_INTERP, OP_PER_NODE = 0, 1
CONV_AUTO, CONV_DIRECT, CONV_FFT = 0, 1, 2
STATUS = {0: "DEBLUR_OK", -1: "DEBLUR_EINVAL", -2: "DEBLUR_ESHAPE", -3: "DEBLUR_ENOMEM", -4: "DEBLUR_ECUDA",
          -5: "DEBLUR_ENCCL", -6: "DEBLUR_ENUMERIC", -7: "DEBLUR_ESTATE"}

_fp = ctypes.POINTER(ctypes.c_float)
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)
_ip = ctypes.POINTER(ctypes.c_int32)


class Params(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("ny", ctypes.c_int64), ("nx", ctypes.c_int64),
        ("psf_gy", ctypes.c_int32), ("psf_gx", ctypes.c_int32), ("psf_size", ctypes.c_int32),
        ("psfs", _fp), ("interp_wy", _fp), ("interp_wx", _fp),
        ("y", _fp), ("noise_w", _fp), ("noise_w_scalar", ctypes.c_float),
        ("lam", ctypes.c_float), ("eps", ctypes.c_float),
        ("reg_kind", ctypes.c_int32), ("tv_boundary", ctypes.c_int32),
        ("gamma", ctypes.c_float), ("rho", ctypes.c_float), ("tau", ctypes.c_double),
        ("inner_steps", ctypes.c_int32),
        ("facet_gy", ctypes.c_int32), ("facet_gx", ctypes.c_int32), ("overlap", ctypes.c_int32),
        ("x0", _fp),
        ("conv_path", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("operator_mode", ctypes.c_int32),
        ("independent", ctypes.c_int32),
        ("local_solver", ctypes.c_int32), ("inner_increment", ctypes.c_int32),
        ("loopback_world", ctypes.c_int32),
    ]


class DeblurError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libdeblur.so (building it in-tree if it is missing)."""
    global _lib
    if _lib is None:
        so = os.environ.get("DEBLUR_LIB_VARIANT")   # A/B measurement of an in-tree build variant
        so = os.path.join(_HERE, so) if so else _SO
        if not os.path.exists(so):
            from . import _build
            _build.build()
        L = ctypes.CDLL(so)
        h = ctypes.c_void_p
        sig = {
            "deblur_nccl_id": ([ctypes.c_void_p], ctypes.c_int),
            "deblur_create": ([ctypes.POINTER(Params), ctypes.POINTER(h)], ctypes.c_int),
            "deblur_destroy": ([h], ctypes.c_int),
            "deblur_apply_H": ([h, _fp, _fp], ctypes.c_int),
            "deblur_apply_HT": ([h, _fp, _fp], ctypes.c_int),
            "deblur_apply_H_device": ([h, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
            "deblur_apply_HT_device": ([h, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
            "deblur_iterate": ([h, ctypes.c_int32], ctypes.c_int),
            "deblur_objective": ([h, _dp], ctypes.c_int),
            "deblur_iterate_traced": ([h, ctypes.c_int32, _dp], ctypes.c_int),
            "deblur_get_image": ([h, _fp], ctypes.c_int),
            "deblur_state_size": ([h, _lp], ctypes.c_int),
            "deblur_get_state": ([h, _fp, _fp], ctypes.c_int),
            "deblur_set_state": ([h, _fp, _fp], ctypes.c_int),
            "deblur_get_outer_iteration": ([h, _ip], ctypes.c_int),
            "deblur_set_outer_iteration": ([h, ctypes.c_int32], ctypes.c_int),
            "deblur_reset": ([h, _fp, _fp], ctypes.c_int),
            "deblur_stage_y": ([h, _fp], ctypes.c_int),
            "deblur_reset_staged": ([h, _fp], ctypes.c_int),
            "deblur_get_image_async": ([h, _fp], ctypes.c_int),
            "deblur_sync": ([h], ctypes.c_int),
            "deblur_get_step": ([h, _dp], ctypes.c_int),
            "deblur_set_profiling": ([h, ctypes.c_int32], ctypes.c_int),
            "deblur_kernel_stats": ([h, _ip, _lp, _dp], ctypes.c_int),
            "deblur_kernel_name": ([ctypes.c_int32], ctypes.c_char_p),
            "deblur_reset_stats": ([h], ctypes.c_int),
            "deblur_kernel_work": ([h, ctypes.c_int32, _dp, _dp], ctypes.c_int),
            "deblur_get_conv_path": ([h, _ip], ctypes.c_int),
            "deblur_get_stream": ([h, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
            "deblur_plan_facets": ([ctypes.POINTER(Params), _ip, _lp, _ip], ctypes.c_int),
            "deblur_plan_messages": ([ctypes.POINTER(Params), ctypes.c_int32, _ip, _lp], ctypes.c_int),
            "deblur_last_error": ([h], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


EXPORTED = ["deblur_nccl_id", "deblur_create", "deblur_destroy", "deblur_apply_H", "deblur_apply_HT",
            "deblur_apply_H_device", "deblur_apply_HT_device", "deblur_iterate", "deblur_iterate_traced",
            "deblur_objective", "deblur_get_image", "deblur_state_size", "deblur_get_state", "deblur_set_state",
            "deblur_get_outer_iteration", "deblur_set_outer_iteration", "deblur_reset",
            "deblur_stage_y", "deblur_reset_staged", "deblur_get_image_async", "deblur_sync",
            "deblur_get_step", "deblur_set_profiling", "deblur_kernel_stats", "deblur_kernel_name",
            "deblur_reset_stats", "deblur_kernel_work", "deblur_get_conv_path", "deblur_get_stream", "deblur_plan_facets", "deblur_plan_messages",
            "deblur_last_error"]


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_fp)


def _check(st: int, handle=None):
    if st != 0:
        msg = lib().deblur_last_error(handle)
        raise DeblurError(st, msg.decode() if msg else "")


def nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().deblur_nccl_id(buf))
    return buf.raw


def make_params(psfs, wy, wx, y, noise_w=None, noise_w_scalar: float = 1.0, lam: float = 0.01,
                eps: float = 1e-3, reg_kind: int = 0, tv_boundary: int = 0, gamma: float = 0.0, rho: float = 1.0,
                tau: float = 0.0, inner_steps: int = 1, facet_gy: int = 1, facet_gx: int = 1, overlap: int = 0,
                x0=None, conv_path: int = CONV_AUTO, rank: int = 0, world: int = 1, device: int = 0,
                nccl_id_bytes: Optional[bytes] = None, operator_mode: int = 0, independent: int = 0,
                local_solver: int = 0, inner_increment: int = 0, loopback_world: int = 0):
    """Returns (Params, keepalive) -- keepalive holds the arrays the pointers refer to."""
    psfs = _f32(psfs)
    wy, wx, y = _f32(wy), _f32(wx), _f32(y)
    K, P, _ = psfs.shape
    gy, ny = wy.shape
    gx, nx = wx.shape
    keep = [psfs, wy, wx, y]
    nw = None
    if noise_w is not None:
        nw = _f32(noise_w)
        keep.append(nw)
    x0a = None
    if x0 is not None:
        x0a = _f32(x0)
        keep.append(x0a)
    idbuf = None
    if nccl_id_bytes is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id_bytes), 128)
        keep.append(idbuf)
    p = Params(abi_version=ABI_VERSION, ny=ny, nx=nx, psf_gy=gy, psf_gx=gx, psf_size=P,
               psfs=_ptr(psfs), interp_wy=_ptr(wy), interp_wx=_ptr(wx), y=_ptr(y), noise_w=_ptr(nw),
               noise_w_scalar=noise_w_scalar, lam=lam, eps=eps, reg_kind=reg_kind, tv_boundary=tv_boundary,
               gamma=gamma, rho=rho, tau=tau, inner_steps=inner_steps, facet_gy=facet_gy, facet_gx=facet_gx,
               overlap=overlap, x0=_ptr(x0a), conv_path=conv_path, rank=rank, world=world, device=device,
               nccl_id=ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
               operator_mode=operator_mode, independent=int(independent), local_solver=local_solver,
               inner_increment=inner_increment, loopback_world=loopback_world)
    return p, keep


def problem_params(pb, **over):
    """make_params for a synth.Problem (same field names)."""
    kw = dict(noise_w=pb.noise_w, noise_w_scalar=pb.noise_w_scalar, lam=pb.lam, eps=pb.eps,
              reg_kind=pb.reg_kind, tv_boundary=pb.tv_boundary, gamma=pb.gamma, rho=pb.rho,
              inner_steps=pb.inner_steps, facet_gy=pb.fy, facet_gx=pb.fx, overlap=pb.overlap, x0=pb.x0,
              operator_mode=getattr(pb, "operator_mode", 0), independent=getattr(pb, "independent", 0),
              local_solver=getattr(pb, "local_solver", 0), inner_increment=getattr(pb, "inner_increment", 0))
    kw.update(over)
    return make_params(pb.psfs, pb.wy, pb.wx, pb.y, **kw)


def plan_facets(params: Params):
    n = ctypes.c_int32(0)
    _check(lib().deblur_plan_facets(ctypes.byref(params), ctypes.byref(n), None, None))
    boxes = np.zeros((n.value, 8), np.int64)
    owner = np.zeros(n.value, np.int32)
    _check(lib().deblur_plan_facets(ctypes.byref(params), ctypes.byref(n), boxes.ctypes.data_as(_lp),
                                    owner.ctypes.data_as(_ip)))
    return boxes, owner


def plan_messages(params: Params, rank: int):
    n = ctypes.c_int32(0)
    _check(lib().deblur_plan_messages(ctypes.byref(params), rank, ctypes.byref(n), None))
    msgs = np.zeros((n.value, 8), np.int64)
    if n.value:
        _check(lib().deblur_plan_messages(ctypes.byref(params), rank, ctypes.byref(n), msgs.ctypes.data_as(_lp)))
    return msgs


class Deblur:
    """One handle = one rank = one GPU (deblur_create ... deblur_destroy)."""

    def __init__(self, params: Params, keepalive=None):
        self._lib = lib()
        self._h = ctypes.c_void_p()
        _check(self._lib.deblur_create(ctypes.byref(params), ctypes.byref(self._h)))
        self.ny, self.nx, self.P = params.ny, params.nx, params.psf_size
        self.my, self.mx = self.ny - self.P + 1, self.nx - self.P + 1
        self.rank = params.rank

    @classmethod
    def from_problem(cls, pb, **over):
        p, keep = problem_params(pb, **over)
        return cls(p, keep)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.deblur_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _c(self, st):
        _check(st, self._h)

    # --- operators -----------------------------------------------------------
    def apply_H(self, x) -> Optional[np.ndarray]:
        x = _f32(x)
        assert x.shape == (self.ny, self.nx)
        out = np.empty((self.my, self.mx), np.float32) if self.rank == 0 else None
        self._c(self._lib.deblur_apply_H(self._h, _ptr(x), _ptr(out)))
        return out

    def apply_HT(self, r) -> Optional[np.ndarray]:
        r = _f32(r)
        assert r.shape == (self.my, self.mx)
        out = np.empty((self.ny, self.nx), np.float32) if self.rank == 0 else None
        self._c(self._lib.deblur_apply_HT(self._h, _ptr(r), _ptr(out)))
        return out

    def apply_H_device(self, d_x: int, d_hx: int):
        self._c(self._lib.deblur_apply_H_device(self._h, ctypes.c_void_p(d_x), ctypes.c_void_p(d_hx)))

    def apply_HT_device(self, d_r: int, d_g: int):
        self._c(self._lib.deblur_apply_HT_device(self._h, ctypes.c_void_p(d_r), ctypes.c_void_p(d_g)))

    # --- solver --------------------------------------------------------------
    def iterate(self, n: int = 1):
        self._c(self._lib.deblur_iterate(self._h, int(n)))
        return self

    def iterate_traced(self, n: int) -> np.ndarray:
        """n iterations; row k = objective (total, data, reg, maxdiff) at x^(k)."""
        out = np.zeros((max(int(n), 0), 4), np.float64)
        self._c(self._lib.deblur_iterate_traced(self._h, int(n), out.ctypes.data_as(_dp)))
        return out

    def objective(self):
        out = (ctypes.c_double * 4)()
        self._c(self._lib.deblur_objective(self._h, out))
        return tuple(out)

    def get_image(self, out: Optional[np.ndarray] = None) -> Optional[np.ndarray]:
        if out is None and self.rank == 0:
            out = np.empty((self.ny, self.nx), np.float32)
        if out is not None:
            assert out.dtype == np.float32 and out.shape == (self.ny, self.nx) and out.flags.c_contiguous
        self._c(self._lib.deblur_get_image(self._h, _ptr(out)))
        return out

    def state_size(self) -> int:
        n = ctypes.c_int64(0)
        self._c(self._lib.deblur_state_size(self._h, ctypes.byref(n)))
        return n.value

    def get_state(self):
        n = self.state_size()
        x = np.empty(n, np.float32) if self.rank == 0 else None
        u = np.empty(n, np.float32) if self.rank == 0 else None
        self._c(self._lib.deblur_get_state(self._h, _ptr(x), _ptr(u)))
        return x, u

    def set_state(self, x, u):
        x, u = _f32(x).ravel(), _f32(u).ravel()
        n = self.state_size()
        if x.size != n or u.size != n:
            raise ValueError(f"set_state: x and u must hold state_size() = {n} floats (got {x.size}, {u.size})")
        self._c(self._lib.deblur_set_state(self._h, _ptr(x), _ptr(u)))

    @property
    def outer_iteration(self) -> int:
        k = ctypes.c_int32(0)
        self._c(self._lib.deblur_get_outer_iteration(self._h, ctypes.byref(k)))
        return k.value

    @outer_iteration.setter
    def outer_iteration(self, k: int):
        self._c(self._lib.deblur_set_outer_iteration(self._h, int(k)))

    def reset(self, y, x0=None):
        y = _f32(y)
        x0 = None if x0 is None else _f32(x0)
        self._c(self._lib.deblur_reset(self._h, _ptr(y), _ptr(x0)))

    # --- pipelined jobs (the caller keeps y / out alive until sync()) ---------------------
    def stage_y(self, y):
        y = np.asarray(y)
        assert y.dtype == np.float32 and y.flags.c_contiguous and y.shape == (self.my, self.mx)
        self._staged_y = y
        self._c(self._lib.deblur_stage_y(self._h, _ptr(y)))

    def reset_staged(self, x0=None):
        x0 = None if x0 is None else _f32(x0)
        self._c(self._lib.deblur_reset_staged(self._h, _ptr(x0)))

    def get_image_async(self, out):
        assert out.dtype == np.float32 and out.shape == (self.ny, self.nx) and out.flags.c_contiguous
        self._c(self._lib.deblur_get_image_async(self._h, _ptr(out)))

    def sync(self):
        self._c(self._lib.deblur_sync(self._h))

    @property
    def tau(self) -> float:
        t = ctypes.c_double(0)
        self._c(self._lib.deblur_get_step(self._h, ctypes.byref(t)))
        return t.value

    @property
    def conv_path(self) -> int:
        p = ctypes.c_int32(0)
        self._c(self._lib.deblur_get_conv_path(self._h, ctypes.byref(p)))
        return p.value

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        self._c(self._lib.deblur_get_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    # --- instrumentation -----------------------------------------------------
    def set_profiling(self, on: bool):
        self._c(self._lib.deblur_set_profiling(self._h, 1 if on else 0))

    def reset_stats(self):
        self._c(self._lib.deblur_reset_stats(self._h))

    def kernel_stats(self):
        n = ctypes.c_int32(64)
        launches = (ctypes.c_int64 * 64)()
        ms = (ctypes.c_double * 64)()
        self._c(self._lib.deblur_kernel_stats(self._h, ctypes.byref(n), launches, ms))
        return {self._lib.deblur_kernel_name(i).decode(): (int(launches[i]), float(ms[i])) for i in range(n.value)}

    def kernel_work(self):
        """{class name: (algorithmic flops, algorithmic bytes) per launch}."""
        out = {}
        i = 0
        while True:
            name = self._lib.deblur_kernel_name(i).decode()
            if not name:
                break
            f, b = ctypes.c_double(0), ctypes.c_double(0)
            self._c(self._lib.deblur_kernel_work(self._h, i, ctypes.byref(f), ctypes.byref(b)))
            out[name] = (f.value, b.value)
            i += 1
        return out
