"""Device context: one mi_ctx per (space-time shape, CUDA device).

PyTorch is used only as plumbing: device memory for vectors, the current
CUDA stream, host<->device copies.  All arithmetic on the (d+1)-way tensors
happens in libmonoiga_b200 kernels.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ExtensionError


def _require_cuda(device):
    if not torch.cuda.is_available():
        raise ExtensionError("a CUDA device is required (no CPU fallback)")
    return torch.device("cuda", device if isinstance(device, int) else torch.device(device).index or 0)


def host_ptr(a):
    """ctypes pointer of a C-contiguous numpy array (kept alive by the caller)."""
    return ctypes.c_void_p(a.ctypes.data)


def dptr(t):
    return ctypes.c_void_p(t.data_ptr())


class DeviceContext:
    """Owns the C context for one space-time shape on one GPU."""

    def __init__(self, space_time, device=0, nt=None, zslab=None):
        """``zslab=(z_lo, z_hi, hz_lo, hz_hi)``: a z-slab context (space-sharded runs) owning the
        global planes [z_lo, z_hi) with hz_lo / hz_hi halo planes on the operator input."""
        self.device = _require_cuda(device)
        st = space_time
        self.space_time = st
        self.d = len(st.spatial)
        self.p = int(st.spatial[0].degree)
        if any(int(s.degree) != self.p for s in st.spatial):
            raise ValueError("all spatial directions must share one degree")
        self.pt = int(st.time.degree)
        self.n = [int(s.dimension) for s in st.spatial]
        self.n3g = self.n[-1]
        self.zslab = None if zslab is None else tuple(int(v) for v in zslab)
        if self.zslab is not None:
            if self.d != 3:
                raise ValueError("z-slab contexts need d = 3")
            self.n[2] = self.zslab[1] - self.zslab[0]
        self.nt = int(st.time.dimension) - 1 if nt is None else int(nt)
        self.ns = int(np.prod(self.n))
        self.N = self.ns * self.nt
        hz = (0, 0) if self.zslab is None else self.zslab[2:]
        self.ns_in = self.ns // self.n[-1] * (self.n[-1] + hz[0] + hz[1])
        self.N_in = self.ns_in * self.nt
        _lib.load()
        h = ctypes.c_void_p()
        dims = np.asarray(self.n, dtype=np.int32)
        with torch.cuda.device(self.device):
            _lib.call("mi_ctx_create", self.device.index, self.d, host_ptr(dims), self.nt, self.p, self.pt,
                      ctypes.byref(h))
        self.handle = h
        if self.zslab is not None:
            z_lo, _, h_lo, h_hi = self.zslab
            _lib.call("mi_ctx_set_zslab", h, z_lo, self.n3g, h_lo, h_hi)
        self._stream = None

    def bind_stream(self):
        """Order library calls on torch's current stream for this device."""
        s = torch.cuda.current_stream(self.device)
        if s is not self._stream:
            _lib.call("mi_ctx_set_stream", self.handle, ctypes.c_void_p(s.cuda_stream))
            self._stream = s
        return s

    def profiling(self, on=True):
        _lib.call("mi_prof_enable", self.handle, 1 if on else 0)

    def read_profile(self, reset=True):
        """{slot: (ms, launches)} accumulated since the last reset."""
        ms = np.zeros(8)
        n = np.zeros(8, dtype=np.int64)
        _lib.call("mi_prof_read", self.handle, host_ptr(ms), host_ptr(n), 1 if reset else 0)
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(_lib.PROF_SLOTS)}

    def close(self):
        if self.handle:
            _lib.load().mi_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64, device=self.device)

    def to_device(self, x):
        """numpy / torch vector -> contiguous fp64 device tensor (flattened)."""
        if isinstance(x, torch.Tensor):
            t = x.to(device=self.device, dtype=torch.float64)
            return t.reshape(-1).contiguous()
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        return torch.from_numpy(a).to(self.device, non_blocking=False)
