"""ctypes binding of libphasemask_b200.so (C ABI in include/phasemask_b200.h).

Loads the in-tree library (building it first when it is missing and nvcc is
available), declares every entry point's signature and maps the library's
error codes onto the exceptions the reference raises. There is no CPU
fallback anywhere: if the library or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PM_LIB", _PKG / "lib" / "libphasemask_b200.so"))

PM_OK = 0
PM_ERR_ARG = -1
PM_ERR_CUDA = -2
PM_ERR_NOMEM = -3
PM_ERR_UNSUPPORTED = -4
PM_ERR_DIVERGED = -5

PM_FORWARD = -1
PM_INVERSE = +1
PM_ALGO_GS = 0
PM_ALGO_RAAR = 1


class pm_params(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int),
        ("beta", C.c_double),
        ("max_iters", C.c_int),
        ("record_every", C.c_int),
        ("early_stop_tol", C.c_double),
        ("t_lit", C.c_double),
        ("t_dark", C.c_double),
        ("p_per_mask", C.c_int),
        ("init_complex", C.c_int),
        ("init_random", C.c_int),
        ("rng", C.c_ulonglong * 4),
    ]


class pm_result(C.Structure):
    _fields_ = [
        ("phases", C.c_void_p),
        ("levels", C.c_void_p),
        ("u_star", C.c_void_p),
        ("v_star", C.c_void_p),
        ("gap", C.c_void_p),
        ("err_lit", C.c_void_p),
        ("err_dark", C.c_void_p),
        ("iters_run", C.c_void_p),
        ("diverged_iter", C.c_void_p),
        ("device_ms", C.c_void_p),
    ]


class pm_record(C.Structure):
    _fields_ = [
        ("gap", C.c_double),
        ("err_lit", C.c_double),
        ("err_dark", C.c_double),
        ("iter", C.c_int),
        ("flags", C.c_int),
    ]


PM_REC_PUBLISHED, PM_REC_RECORDED, PM_REC_EARLY, PM_REC_DIVERGED, PM_REC_STOP, PM_REC_ABORTED = 1, 2, 4, 8, 16, 32
PM_REC_TIMEOUT = 64


# name -> (restype, argtypes); mirrors include/phasemask_b200.h one to one
_VP, _I, _D, _LL = C.c_void_p, C.c_int, C.c_double, C.c_longlong
SIGNATURES = {
    "pm_version": (_I, []),
    "pm_device_count": (_I, [C.POINTER(_I)]),
    "pm_last_error": (C.c_char_p, []),
    "pm_plan_create": (_I, [_I, _I, _I, _I, _I, C.POINTER(_VP)]),
    "pm_plan_destroy": (_I, [_VP]),
    "pm_plan_set_stream": (_I, [_VP, _VP]),
    "pm_plan_get_stream": (_I, [_VP, C.POINTER(_VP)]),
    "pm_plan_synchronize": (_I, [_VP]),
    "pm_plan_launch_count": (_I, [_VP, C.POINTER(_LL)]),
    "pm_plan_set_path": (_I, [_VP, _I]),
    "pm_plan_get_path": (_I, [_VP, C.POINTER(_I)]),
    "pm_fft2": (_I, [_VP, _VP, _VP, _I, _I]),
    "pm_fft2_device": (_I, [_VP, _VP, _VP, _I, _I]),
    "pm_replace_modulus": (_I, [_VP, _VP, _VP, _I, _D, _VP, _I]),
    "pm_replace_modulus_device": (_I, [_VP, _VP, _VP, _I, _D, _VP, _I]),
    "pm_project_fourier": (_I, [_VP, _VP, _VP, _D, _VP]),
    "pm_gap": (_I, [_VP, _VP, _VP, _VP, _D, _D, C.POINTER(_D)]),
    "pm_norm2": (_I, [_I, _VP, _LL, _I, C.POINTER(_D)]),
    "pm_sum": (_I, [_I, _VP, _LL, C.POINTER(_D)]),
    "pm_phases": (_I, [_I, _VP, _LL, _I, _D, _VP]),
    "pm_naive_dft": (_I, [_I, _VP, _I, _I, _I, _VP]),
    "pm_random_start": (_I, [_I, _VP, _LL, _I, _I, _VP, _VP]),
    "pm_recon_image": (_I, [_VP, _VP, _I, _VP, _D, _VP, _VP]),
    "pm_solve": (_I, [_VP, _VP, _VP, _VP, _I, C.POINTER(pm_params), _VP, _VP, _VP,
                      C.POINTER(pm_result)]),
    "pm_solve_device": (_I, [_VP, _VP, _VP, _VP, _I, C.POINTER(pm_params), _VP, _VP, _VP,
                             C.POINTER(pm_result)]),
    "pm_solve_begin": (_I, [_VP, _VP, _VP, _VP, _I, C.POINTER(pm_params), _VP, _VP, _VP]),
    "pm_solve_step": (_I, [_VP, _I, C.POINTER(_I)]),
    "pm_solve_records": (_I, [_VP, _I, _I, _VP, _VP, _VP, _VP, _VP]),
    "pm_solve_finish": (_I, [_VP, _I, C.POINTER(pm_result)]),
    "pm_solve_async": (_I, [_VP, _VP, _VP, _VP, C.POINTER(pm_params), _VP, _VP, _VP, _I, C.POINTER(pm_result)]),
    "pm_solve_next": (_I, [_VP, _I, C.POINTER(pm_record)]),
    "pm_solve_answer": (_I, [_VP, _I, _I]),
    "pm_solve_wait": (_I, [_VP, C.POINTER(pm_result)]),
    "pm_time_sweep": (_I, [_VP, _I, _I, _I, C.POINTER(C.c_float)]),
    "pm_measure_copy": (_I, [_I, _LL, _I, C.POINTER(_D)]),
    "pm_measure_l2": (_I, [_I, _LL, _I, _I, C.POINTER(_D)]),
    "pm_host_alloc": (_I, [_LL, C.POINTER(_VP)]),
    "pm_host_free": (_I, [_VP]),
    "pm_debug_phase_stamps": (_I, [_VP, _I, _VP, _I]),
}

_lib = None
_lock = threading.Lock()


class SolveDivergedFromLib(RuntimeError):
    """Internal: the library reported non-finite values (PM_ERR_DIVERGED)."""


def load(build_if_missing: bool = True):
    """Load (and, if needed, build) the native library; raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if not build_if_missing or os.environ.get("PM_NO_AUTOBUILD"):
                raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_1302_0120_b200.build`")
            from .build import build
            build()
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().pm_last_error().decode(errors="replace")


def check(code: int, what: str = ""):
    """Map a PM_ERR_* code to the reference's exception types."""
    if code == PM_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if code == PM_ERR_ARG:
        raise ValueError(msg)
    if code == PM_ERR_NOMEM:
        raise MemoryError(msg)
    if code == PM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if code == PM_ERR_DIVERGED:
        raise SolveDivergedFromLib(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    n = C.c_int(0)
    check(load().pm_device_count(C.byref(n)))
    return n.value


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- plans

class Plan:
    """Owns one pm_plan: a grid, a precision, device buffers and a stream.

    The analogue of the reference's FftProvider / PlanCache entry
    (src/transform.py:23-35, src/service.py:65-82). Thread-safe: calls are
    serialised by a per-plan lock, as PlanCache does.
    """

    def __init__(self, n_x: int, n_y: int, precision_code: int, device: int = 0, max_batch: int = 1):
        self.lib = load()
        self.n_x, self.n_y, self.prec, self.device = n_x, n_y, precision_code, device
        self.lock = threading.Lock()
        h = C.c_void_p()
        check(self.lib.pm_plan_create(device, n_x, n_y, precision_code, max_batch, C.byref(h)),
              "pm_plan_create")
        self.handle = h

    @property
    def complex_dtype(self):
        return np.complex64 if self.prec == 0 else np.complex128

    @property
    def float_dtype(self):
        return np.float32 if self.prec == 0 else np.float64

    def close(self):
        if getattr(self, "handle", None):
            self.lib.pm_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self) -> int:
        n = C.c_longlong(0)
        check(self.lib.pm_plan_launch_count(self.handle, C.byref(n)))
        return n.value

    def set_path(self, path: int):
        """0 auto, 1 persistent cooperative kernel, 2 sweep-per-kernel graph."""
        check(self.lib.pm_plan_set_path(self.handle, path), "pm_plan_set_path")

    def path(self) -> int:
        v = C.c_int(0)
        check(self.lib.pm_plan_get_path(self.handle, C.byref(v)))
        return v.value

    def set_stream(self, stream_handle: int | None):
        check(self.lib.pm_plan_set_stream(self.handle, C.c_void_p(stream_handle or 0)))

    def synchronize(self):
        check(self.lib.pm_plan_synchronize(self.handle))

    # ---- transforms / projections (host arrays)
    def fft2(self, data: np.ndarray, direction: int) -> np.ndarray:
        x = np.ascontiguousarray(data, dtype=self.complex_dtype)
        batch = 1 if x.ndim == 2 else x.shape[0]
        out = np.empty_like(x)
        with self.lock:
            check(self.lib.pm_fft2(self.handle, ptr(x), ptr(out), direction, batch), "pm_fft2")
        return out

    def replace_modulus(self, data: np.ndarray, target: np.ndarray, zero_tol: float) -> np.ndarray:
        x = np.ascontiguousarray(data, dtype=self.complex_dtype)
        t = np.ascontiguousarray(target, dtype=self.float_dtype)
        batch = 1 if x.ndim == 2 else x.shape[0]
        per_field = int(t.ndim == 3)
        out = np.empty_like(x)
        with self.lock:
            check(self.lib.pm_replace_modulus(self.handle, ptr(x), ptr(t), per_field,
                                              float(zero_tol), ptr(out), batch), "pm_replace_modulus")
        return out

    def project_fourier(self, u: np.ndarray, m: np.ndarray, tol_m: float) -> np.ndarray:
        x = np.ascontiguousarray(u, dtype=self.complex_dtype)
        t = np.ascontiguousarray(m, dtype=self.float_dtype)
        out = np.empty_like(x)
        with self.lock:
            check(self.lib.pm_project_fourier(self.handle, ptr(x), ptr(t), float(tol_m), ptr(out)),
                  "pm_project_fourier")
        return out

    def gap(self, u, p, m, tol_p, tol_m) -> float:
        x = np.ascontiguousarray(u, dtype=self.complex_dtype)
        pp = np.ascontiguousarray(p, dtype=self.float_dtype)
        mm = np.ascontiguousarray(m, dtype=self.float_dtype)
        g = C.c_double(0.0)
        with self.lock:
            check(self.lib.pm_gap(self.handle, ptr(x), ptr(pp), ptr(mm), float(tol_p), float(tol_m),
                                  C.byref(g)), "pm_gap")
        return g.value

    def recon_image(self, u, target_energy=None, log_floor=None, intensity=True):
        """(intensity or None, log image or None) of pm_recon_image for a
        (n_y, n_x) field or a (B, n_y, n_x) stack; target_energy: scalar or
        per-field array (None: unscaled)."""
        x = np.ascontiguousarray(u, dtype=self.complex_dtype)
        shape = x.shape
        batch = x.size // (shape[-1] * shape[-2])
        en = None if target_energy is None else np.ascontiguousarray(
            np.broadcast_to(np.asarray(target_energy, dtype=np.float64), (batch,)))
        inten = np.empty(shape, dtype=np.float64) if intensity else None
        img = np.empty(shape, dtype=np.uint8) if log_floor is not None else None
        with self.lock:
            check(self.lib.pm_recon_image(self.handle, ptr(x), batch, ptr(en),
                                          float(log_floor or 0.0), ptr(img), ptr(inten)),
                  "pm_recon_image")
        return inten, img

    def time_sweep(self, which: int, batch: int, reps: int) -> float:
        ms = C.c_float(0)
        with self.lock:
            check(self.lib.pm_time_sweep(self.handle, which, batch, reps, C.byref(ms)), "pm_time_sweep")
        return float(ms.value)


# ---------------------------------------------------------- plan-less helpers

_DTYPE_CODE = {np.dtype(np.float32): 0, np.dtype(np.float64): 1,
               np.dtype(np.complex64): 2, np.dtype(np.complex128): 3}


def norm2(data: np.ndarray, device: int = 0) -> float:
    a = np.ascontiguousarray(data)
    if a.dtype not in _DTYPE_CODE:
        a = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    out = C.c_double(0.0)
    check(load().pm_norm2(device, ptr(a), a.size, _DTYPE_CODE[a.dtype], C.byref(out)), "pm_norm2")
    return out.value


def fixed_sum(values: np.ndarray, device: int = 0) -> float:
    a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    out = C.c_double(0.0)
    check(load().pm_sum(device, ptr(a), a.size, C.byref(out)), "pm_sum")
    return out.value


def phases(u: np.ndarray, zero_tol: float = 0.0, device: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(u)
    if a.dtype not in (np.complex64, np.complex128):
        a = a.astype(np.complex128)
    prec = 0 if a.dtype == np.complex64 else 1
    out = np.empty(a.shape, dtype=np.float64)
    check(load().pm_phases(device, ptr(a), a.size, prec, float(zero_tol), ptr(out)), "pm_phases")
    return out


def naive_dft(data: np.ndarray, direction: int, device: int = 0) -> np.ndarray:
    """Dense fp64 unitary DFT of a (n_y, n_x) array on the device (pm_naive_dft)."""
    a = np.ascontiguousarray(data, dtype=np.complex128)
    out = np.empty_like(a)
    check(load().pm_naive_dft(device, ptr(a), a.shape[1], a.shape[0], direction, ptr(out)), "pm_naive_dft")
    return out


def pcg64_state(seed: int) -> np.ndarray:
    """The PCG64 state {state hi, lo, inc hi, lo} of np.random.default_rng(seed)
    right after seeding (SeedSequence hashing stays on the host)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m64 = (1 << 64) - 1
    return np.array([st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64],
                    dtype=np.uint64)


def random_start(m: np.ndarray, complex_dtype, seed: int, device: int = 0) -> np.ndarray:
    """m e^{i phi} with phi = default_rng(seed).uniform(0, 2 pi, m.shape[-2:])
    drawn on the device (pm_random_start); m is (n_y, n_x) or a (B, n_y, n_x)
    stack sharing the draws."""
    prec = 0 if np.dtype(complex_dtype) == np.complex64 else 1
    a = np.ascontiguousarray(m, dtype=np.float32 if prec == 0 else np.float64)
    count = a.shape[-1] * a.shape[-2]
    batch = a.size // count
    out = np.empty(a.shape, dtype=complex_dtype)
    rng = pcg64_state(seed)
    check(load().pm_random_start(device, ptr(a), count, batch, prec, ptr(rng), ptr(out)),
          "pm_random_start")
    return out


def measure_copy(nbytes: int, reps: int = 10, device: int = 0) -> float:
    g = C.c_double(0.0)
    check(load().pm_measure_copy(device, int(nbytes), reps, C.byref(g)), "pm_measure_copy")
    return g.value


def measure_l2(nbytes: int, passes: int = 50, mode: int = 1, device: int = 0) -> float:
    """L2-resident bandwidth in GB/s (mode 1: copy, read + write bytes; 0: reads)."""
    v = C.c_double(0.0)
    check(load().pm_measure_l2(device, nbytes, passes, mode, C.byref(v)), "pm_measure_l2")
    return v.value


class _PinnedPool:
    """Page-locked host buffers from the library's own CUDA runtime
    (pm_host_alloc). Memory pinned by another runtime in the process (torch's
    caching host allocator) is not recognised as pinned by the library's
    copies, which then run at pageable speed; these buffers are. A dropped
    array's block returns to a per-size free list (bounded)."""

    MAX_CACHED = 1 << 30

    def __init__(self):
        self.free: dict[int, list[int]] = {}
        self.cached = 0
        # re-entrant: a finaliser (returning a block) may run while this thread holds it
        self.lock = threading.RLock()

    def _release(self, size: int, ptr: int):
        with self.lock:
            if self.cached + size <= self.MAX_CACHED:
                self.free.setdefault(size, []).append(ptr)
                self.cached += size
                return
        try:
            load().pm_host_free(C.c_void_p(ptr))
        except Exception:                        # interpreter shutdown: the process frees it
            pass

    def empty(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        size = max(4096, (n + 65535) & ~65535)
        with self.lock:
            lst = self.free.get(size)
            ptr = lst.pop() if lst else None
            if ptr is not None:
                self.cached -= size
        if ptr is None:
            out = C.c_void_p(0)
            check(load().pm_host_alloc(size, C.byref(out)), "pm_host_alloc")
            ptr = out.value
        buf = (C.c_ubyte * size).from_address(ptr)
        weakref.finalize(buf, self._release, size, ptr)
        return np.frombuffer(buf, dtype=np.uint8, count=n).view(dtype).reshape(shape)


_pool = _PinnedPool()


def host_empty(shape, dtype) -> np.ndarray:
    """An uninitialised C-contiguous array in page-locked memory the library
    copies from / to at full speed (pass such arrays to the batch API)."""
    return _pool.empty(shape, dtype)
