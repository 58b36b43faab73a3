"""Device memory without torch: the CUDA runtime that libaffmae_b200.so links
(libcudart.so.12, resolved through the already-loaded library) via ctypes.  Plumbing for
the torch-free host path (model.py, the `_affmae` module): allocations, pinned host
buffers, copies, streams and events."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi

_rt = None
H2D, D2H, D2D = 1, 2, 3


def rt():
    global _rt
    if _rt is None:
        capi.lib()  # loads libcudart.so.12 as a dependency first
        _rt = C.CDLL("libcudart.so.12")
        for f in ("cudaMalloc", "cudaFree", "cudaMemcpy", "cudaMemcpyAsync", "cudaMemsetAsync",
                  "cudaStreamSynchronize", "cudaDeviceSynchronize", "cudaStreamCreate", "cudaStreamDestroy",
                  "cudaEventCreate", "cudaEventRecord", "cudaEventSynchronize", "cudaEventElapsedTime",
                  "cudaEventDestroy", "cudaMallocHost", "cudaFreeHost", "cudaGetErrorString", "cudaSetDevice"):
            getattr(_rt, f).restype = C.c_int if f != "cudaGetErrorString" else C.c_char_p
    return _rt


def _ok(rc, what):
    if rc != 0:
        raise capi.AffmaeError(f"{what}: {rt().cudaGetErrorString(rc).decode()}")


class DeviceBuffer:
    def __init__(self, nbytes: int):
        p = C.c_void_p()
        _ok(rt().cudaMalloc(C.byref(p), C.c_size_t(max(int(nbytes), 1))), "cudaMalloc")
        self.ptr, self.nbytes = p.value, int(nbytes)

    def free(self):
        if getattr(self, "ptr", None):
            rt().cudaFree(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory viewed as a numpy array."""

    def __init__(self, shape, dtype):
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        _ok(rt().cudaMallocHost(C.byref(p), C.c_size_t(max(n, 1))), "cudaMallocHost")
        self.ptr = p.value
        self.array = np.ctypeslib.as_array((C.c_uint8 * max(n, 1)).from_address(self.ptr))[:n].view(dt).reshape(shape)

    def free(self):
        if getattr(self, "ptr", None):
            rt().cudaFreeHost(C.c_void_p(self.ptr))
            self.ptr = None


def h2d(dst_ptr: int, a: np.ndarray, stream=None):
    a = np.ascontiguousarray(a)
    if stream is None:
        _ok(rt().cudaMemcpy(C.c_void_p(dst_ptr), a.ctypes.data_as(C.c_void_p), C.c_size_t(a.nbytes), H2D), "h2d")
    else:
        _ok(rt().cudaMemcpyAsync(C.c_void_p(dst_ptr), a.ctypes.data_as(C.c_void_p), C.c_size_t(a.nbytes), H2D,
                                 C.c_void_p(stream)), "h2d")
        sync(stream)


def h2d_async(dst_ptr: int, src_ptr: int, nbytes: int, stream):
    _ok(rt().cudaMemcpyAsync(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), C.c_size_t(nbytes), H2D, C.c_void_p(stream)),
        "h2d_async")


def d2h_async(dst_ptr: int, src_ptr: int, nbytes: int, stream):
    _ok(rt().cudaMemcpyAsync(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), C.c_size_t(nbytes), D2H, C.c_void_p(stream)),
        "d2h_async")


def d2d_async(dst_ptr: int, src_ptr: int, nbytes: int, stream):
    _ok(rt().cudaMemcpyAsync(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), C.c_size_t(nbytes), 3, C.c_void_p(stream)),
        "d2d_async")  # cudaMemcpyDeviceToDevice


def stream_wait(stream, event: "Event"):
    """`stream` waits for the work recorded in `event`."""
    _ok(rt().cudaStreamWaitEvent(C.c_void_p(stream), event.e, 0), "cudaStreamWaitEvent")


def d2h(src_ptr: int, shape, dtype, stream=None) -> np.ndarray:
    out = np.empty(shape, dtype)
    if stream is not None:
        sync(stream)
    _ok(rt().cudaMemcpy(out.ctypes.data_as(C.c_void_p), C.c_void_p(src_ptr), C.c_size_t(out.nbytes), D2H), "d2h")
    return out


def sync(stream=None):
    if stream is None:
        _ok(rt().cudaDeviceSynchronize(), "cudaDeviceSynchronize")
    else:
        _ok(rt().cudaStreamSynchronize(C.c_void_p(stream)), "cudaStreamSynchronize")


def stream_create() -> int:
    s = C.c_void_p()
    _ok(rt().cudaStreamCreate(C.byref(s)), "cudaStreamCreate")
    return s.value


class Event:
    def __init__(self):
        e = C.c_void_p()
        _ok(rt().cudaEventCreate(C.byref(e)), "cudaEventCreate")
        self.e = e

    def record(self, stream=None):
        _ok(rt().cudaEventRecord(self.e, C.c_void_p(stream)), "cudaEventRecord")

    def synchronize(self):
        _ok(rt().cudaEventSynchronize(self.e), "cudaEventSynchronize")

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        _ok(rt().cudaEventElapsedTime(C.byref(ms), self.e, end.e), "cudaEventElapsedTime")
        return float(ms.value)
