"""Thin ctypes binding of libfbp (include/fbp.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module never computes anything itself and has no CPU fallback: if libfbp.so is
missing or the device is not an sm_100 B200 it raises.

    plan = Plan(n=2048, b=[...], a=[...], max_batch=64, device=0)
    img  = plan.reconstruct(sino)            # sino: float32 cuda [B, 4, N, 2N]
    F    = plan.iir_filter(sino)             # Eq.12-13
    bp   = plan.backproject(F, scale=1/N)    # Eq.19-22
    lin  = plan.forward(img)                 # Eq.17 (forward FHT)
    lin  = plan.resample(sino_rtheta, dr=1)  # Eq.14-15 (scanner sinogram -> linogram)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfbp.so")
_lib = None

FBP_STATUS = {0: "FBP_OK", 1: "FBP_ERR_PLAN", 2: "FBP_ERR_PARAM", 3: "FBP_ERR_UNSTABLE",
              4: "FBP_ERR_CUDA", 5: "FBP_ERR_NOMEM", 6: "FBP_ERR_DEVICE"}

EXPORTED = ["fbp_plan_create", "fbp_plan_destroy", "fbp_iir_filter", "fbp_fht_backproject",
            "fbp_fht_forward", "fbp_resample_sinogram", "fbp_reconstruct", "fbp_reconstruct_host", "fbp_status_str", "fbp_last_error",
            "fbp_plan_launch_count", "fbp_plan_info", "fbp_plan_path", "fbp_plan_profile",
            "fbp_plan_kernel_times"]

KERNEL_KINDS = ("iir", "fht_pass_a", "fht_pass_b", "fwd_pass_a", "fwd_pass_b", "resample", "small")


class FbpError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{FBP_STATUS.get(status, status)}: {detail}")
        self.status = status


def lib():
    """Load libfbp.so (built in-tree by paper_2007_06289_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_2007_06289_b200.build`")
    L = ctypes.CDLL(_LIB_PATH)
    vp, i, f, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.POINTER(ctypes.c_double)
    L.fbp_plan_create.argtypes = [ctypes.POINTER(vp), i, i, i, d, i, d, i]
    L.fbp_plan_create.restype = i
    L.fbp_plan_destroy.argtypes = [vp]
    L.fbp_plan_destroy.restype = None
    L.fbp_iir_filter.argtypes = [vp, vp, vp, i, vp]
    L.fbp_iir_filter.restype = i
    L.fbp_fht_backproject.argtypes = [vp, vp, vp, i, f, vp]
    L.fbp_fht_backproject.restype = i
    L.fbp_fht_forward.argtypes = [vp, vp, vp, i, vp]
    L.fbp_fht_forward.restype = i
    L.fbp_resample_sinogram.argtypes = [vp, vp, i, i, ctypes.c_double, vp, i, vp]
    L.fbp_resample_sinogram.restype = i
    L.fbp_reconstruct.argtypes = [vp, vp, vp, i, vp]
    L.fbp_reconstruct.restype = i
    L.fbp_reconstruct_host.argtypes = [vp, vp, vp, i]
    L.fbp_reconstruct_host.restype = i
    L.fbp_status_str.argtypes = [i]
    L.fbp_status_str.restype = ctypes.c_char_p
    L.fbp_last_error.argtypes = []
    L.fbp_last_error.restype = ctypes.c_char_p
    L.fbp_plan_launch_count.argtypes = [vp]
    L.fbp_plan_launch_count.restype = ctypes.c_longlong
    L.fbp_plan_info.argtypes = [vp] + [ctypes.POINTER(i)] * 4 + [ctypes.POINTER(ctypes.c_longlong)]
    L.fbp_plan_info.restype = i
    L.fbp_plan_path.argtypes = [vp] + [ctypes.POINTER(i)] * 3
    L.fbp_plan_path.restype = i
    L.fbp_plan_profile.argtypes = [vp, i]
    L.fbp_plan_profile.restype = i
    L.fbp_plan_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_longlong), i]
    L.fbp_plan_kernel_times.restype = i
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise FbpError(status, lib().fbp_last_error().decode())


def _stream_ptr(stream, device: int) -> int:
    """The caller's stream, else the current stream of the plan's device."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    if s.device.index != device:
        raise ValueError(f"stream is on cuda:{s.device.index}, the plan on cuda:{device}")
    return s.cuda_stream


class Plan:
    """fbp_plan: N, IIR coefficients (Eq.9 sign), workspace on one device."""

    def __init__(self, n: int, b, a, max_batch: int = 1, device: int = 0):
        L = lib()
        self.n = int(n)
        self.b = [float(v) for v in b]
        self.a = [float(v) for v in a]
        self.max_batch = int(max_batch)
        self.device = int(device)
        bb = (ctypes.c_double * max(1, len(self.b)))(*self.b)
        aa = (ctypes.c_double * max(1, len(self.a)))(*self.a)
        h = ctypes.c_void_p()
        _check(L.fbp_plan_create(ctypes.byref(h), self.n, self.max_batch, len(self.b), bb,
                                 len(self.a), aa, self.device))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fbp_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- info
    def info(self) -> dict:
        n, k1, m, grp = (ctypes.c_int() for _ in range(4))
        ws = ctypes.c_longlong()
        _check(lib().fbp_plan_info(self._h, ctypes.byref(n), ctypes.byref(k1), ctypes.byref(m),
                                   ctypes.byref(grp), ctypes.byref(ws)))
        return dict(N=n.value, k1=k1.value, m=m.value, group=grp.value, workspace_bytes=ws.value)

    def path(self) -> dict:
        """Schedule: fused sweep fast path or the separate-kernel path (fbp_plan_path)."""
        fast, d, x = (ctypes.c_int() for _ in range(3))
        _check(lib().fbp_plan_path(self._h, ctypes.byref(fast), ctypes.byref(d), ctypes.byref(x)))
        return dict(fast=bool(fast.value), lookahead_tiles=d.value, tile_width=x.value)

    def launch_count(self) -> int:
        """Kernels launched by the last call on this plan."""
        return int(lib().fbp_plan_launch_count(self._h))

    def profile(self, enable: bool = True):
        """Enable (and clear) / disable per-kernel CUDA-event timing inside libfbp."""
        _check(lib().fbp_plan_profile(self._h, int(bool(enable))))

    def kernel_times(self) -> dict:
        """{kind: (total_ms, launches)} since the last profile(True); clears the record."""
        k = len(KERNEL_KINDS)
        ms = (ctypes.c_double * k)()
        n = (ctypes.c_longlong * k)()
        _check(lib().fbp_plan_kernel_times(self._h, ms, n, k))
        return {k: (ms[i], n[i]) for i, k in enumerate(KERNEL_KINDS)}

    # ------------------------------------------------------------- checks
    def _dev(self, x: torch.Tensor, name: str):
        if x.device.index != self.device:
            raise ValueError(f"{name} is on {x.device}, the plan on cuda:{self.device}")

    def _lin(self, x: torch.Tensor, name: str, batch: int | None = None) -> torch.Tensor:
        N = self.n
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32):
            raise TypeError(f"{name} must be a float32 CUDA tensor")
        self._dev(x, name)
        if x.dim() == 3:
            x = x.unsqueeze(0)
        if tuple(x.shape[1:]) != (4, N, 2 * N):
            raise ValueError(f"{name} must have shape [B, 4, {N}, {2 * N}], got {tuple(x.shape)}")
        if not x.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if batch is not None and x.shape[0] != batch:
            raise ValueError(f"{name} has batch {x.shape[0]}, the input {batch}")
        return x

    def _img_out(self, out, B):
        N = self.n
        if out is None:
            return torch.empty((B, N, N), device=f"cuda:{self.device}", dtype=torch.float32)
        if (not isinstance(out, torch.Tensor) or not out.is_cuda or tuple(out.shape) != (B, N, N)
                or out.dtype != torch.float32 or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous float32 CUDA [{B}, {N}, {N}] tensor")
        self._dev(out, "out")
        return out

    # ---------------------------------------------------------------- ops
    def iir_filter(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        x = self._lin(sino, "sino")
        out = torch.empty_like(x) if out is None else self._lin(out, "out", x.shape[0])
        _check(lib().fbp_iir_filter(self._h, x.data_ptr(), out.data_ptr(), x.shape[0],
                                    _stream_ptr(stream, self.device)))
        return out

    def backproject(self, lin: torch.Tensor, scale: float = 1.0, out: torch.Tensor | None = None,
                    stream=None):
        x = self._lin(lin, "lin")
        out = self._img_out(out, x.shape[0])
        _check(lib().fbp_fht_backproject(self._h, x.data_ptr(), out.data_ptr(), x.shape[0],
                                         float(scale), _stream_ptr(stream, self.device)))
        return out

    def forward(self, image: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """Forward dyadic projection (Eq.17), image [B, N, N] -> linogram [B, 4, N, 2N]."""
        N = self.n
        if not (isinstance(image, torch.Tensor) and image.is_cuda and image.dtype == torch.float32):
            raise TypeError("image must be a float32 CUDA tensor")
        if image.dim() == 2:
            image = image.unsqueeze(0)
        if tuple(image.shape[1:]) != (N, N) or not image.is_contiguous():
            raise ValueError(f"image must be a contiguous [B, {N}, {N}] tensor, got {tuple(image.shape)}")
        self._dev(image, "image")
        B = image.shape[0]
        if out is None:
            out = torch.empty((B, 4, N, 2 * N), device=image.device, dtype=torch.float32)
        else:
            out = self._lin(out, "out", B)
        _check(lib().fbp_fht_forward(self._h, image.data_ptr(), out.data_ptr(), B,
                                     _stream_ptr(stream, self.device)))
        return out

    def resample(self, sino: torch.Tensor, dr: float = 1.0, out: torch.Tensor | None = None, stream=None):
        """Scanner sinogram [B, n_angles, n_bins] -> linogram [B, 4, N, 2N] (Eq.14-15)."""
        N = self.n
        if not (isinstance(sino, torch.Tensor) and sino.is_cuda and sino.dtype == torch.float32):
            raise TypeError("sino must be a float32 CUDA tensor")
        if sino.dim() == 2:
            sino = sino.unsqueeze(0)
        if sino.dim() != 3 or not sino.is_contiguous():
            raise ValueError(f"sino must be a contiguous [B, n_angles, n_bins] tensor, got {tuple(sino.shape)}")
        self._dev(sino, "sino")
        B, na, nb = sino.shape
        if out is None:
            out = torch.empty((B, 4, N, 2 * N), device=sino.device, dtype=torch.float32)
        else:
            out = self._lin(out, "out", B)
        _check(lib().fbp_resample_sinogram(self._h, sino.data_ptr(), na, nb, float(dr), out.data_ptr(), B,
                                           _stream_ptr(stream, self.device)))
        return out

    def reconstruct(self, sino: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        x = self._lin(sino, "sino")
        out = self._img_out(out, x.shape[0])
        _check(lib().fbp_reconstruct(self._h, x.data_ptr(), out.data_ptr(), x.shape[0],
                                     _stream_ptr(stream, self.device)))
        return out

    def reconstruct_host(self, sino, out=None):
        """Host buffers in, host buffers out (numpy or CPU torch, float32, contiguous).

        Synchronous.  `out` (if given) must be a contiguous float32 host buffer of
        shape [B, N, N] of the same kind as `sino`: the library writes B*N*N floats
        into it.  Not thread-safe per plan: one host thread per plan."""
        N = self.n
        want = (4, N, 2 * N)
        if isinstance(sino, torch.Tensor):
            if sino.is_cuda or sino.dtype != torch.float32 or not sino.is_contiguous():
                raise TypeError("sino must be a contiguous float32 CPU tensor")
            if sino.dim() != 4 or tuple(sino.shape[1:]) != want:
                raise ValueError(f"sino must have shape [B, 4, {N}, {2 * N}], got {tuple(sino.shape)}")
            B = sino.shape[0]
            if out is None:
                out = torch.empty((B, N, N), dtype=torch.float32, pin_memory=sino.is_pinned())
            elif (not isinstance(out, torch.Tensor) or out.is_cuda or out.dtype != torch.float32
                  or not out.is_contiguous() or tuple(out.shape) != (B, N, N)):
                raise ValueError(f"out must be a contiguous float32 CPU tensor of shape [{B}, {N}, {N}]")
            ptr_in, ptr_out = sino.data_ptr(), out.data_ptr()
        else:
            sino = np.ascontiguousarray(sino, dtype=np.float32)
            if sino.ndim != 4 or tuple(sino.shape[1:]) != want:
                raise ValueError(f"sino must have shape [B, 4, {N}, {2 * N}], got {tuple(sino.shape)}")
            B = sino.shape[0]
            if out is None:
                out = np.empty((B, N, N), dtype=np.float32)
            elif (not isinstance(out, np.ndarray) or out.dtype != np.float32
                  or not out.flags["C_CONTIGUOUS"] or not out.flags["WRITEABLE"] or out.shape != (B, N, N)):
                raise ValueError(f"out must be a writeable C-contiguous float32 array of shape [{B}, {N}, {N}]")
            ptr_in, ptr_out = sino.ctypes.data, out.ctypes.data
        _check(lib().fbp_reconstruct_host(self._h, ptr_in, ptr_out, B))
        return out
