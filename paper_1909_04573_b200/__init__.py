"""paper_1909_04573_b200 — B200 (sm_100a) hot path of SDA-frame PRNU fingerprint
extraction (Taspinar, Mohanty, Memon, arXiv 1909.04573).

A thin ctypes binding over ``libprnu.so`` (C ABI in ``include/prnu.h``).  This
module only marshals arguments: it checks tensors, allocates outputs and
workspaces with torch (device memory + the current CUDA stream), and calls
the C entry points of the same name.  Every step of the path runs in the
library's CUDA kernels; there is no CPU fallback, and importing fails loudly
if the library has not been built (``python __graft_entry__.py`` or
``paper_1909_04573_b200._build.build()``).

Citations: P:<n> = PAPER.md line, S:<n> = SPEC.md line, R-<n> = DESIGN.md reading.
"""
from __future__ import annotations

import ctypes
import functools
import os
import re
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libprnu.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "prnu.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                      "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PLANE_TOO_SMALL", 3: "DEPTH_EXCEEDS_FRAMES", 4: "BAD_PARAMETER",
          5: "DIMENSION_MISMATCH", 6: "EMPTY_ACCUMULATOR", 7: "CONSTANT_INPUT", 8: "DEGENERATE_SURFACE",
          9: "WORKSPACE_TOO_SMALL", 10: "CUDA_ERROR"}
PCE_THRESHOLD = 60.0   # P:259, strict ">"


class PrnuError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = _lib.prnu_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(code, code)} ({msg})")
        self.code = code


class _Params(ctypes.Structure):
    _fields_ = [("sigma0_sq", ctypes.c_float), ("levels", ctypes.c_int), ("n_windows", ctypes.c_int),
                ("windows", ctypes.c_int * 4)]


@dataclass
class DenoiseParams:
    """Parameters of F (R-1..R-8): sigma0^2 = 9, 4 levels, windows {3,5,7,9}."""
    sigma0_sq: float = 9.0
    levels: int = 4
    windows: tuple = field(default=(3, 5, 7, 9))

    def c(self) -> _Params:
        p = _Params()
        p.sigma0_sq = float(self.sigma0_sq)
        p.levels = int(self.levels)
        p.n_windows = len(self.windows)
        for i, w in enumerate(self.windows[:4]):
            p.windows[i] = int(w)
        return p


class _Variant(ctypes.Structure):
    _fields_ = [("taps", ctypes.c_int), ("boundary", ctypes.c_int), ("transform", ctypes.c_int)]


@dataclass
class DenoiseVariant:
    """f3 denoiser variant (R-24..R-26; include/prnu.h): taps 8 or 16 (db8),
    boundary 0 (half-sample symmetric) or 1 (pad + periodic), transform 0 (decimated) or
    1 (undecimated; circular, so boundary must be 1)."""
    taps: int = 8
    boundary: int = 0
    transform: int = 0

    def c(self) -> _Variant:
        v = _Variant()
        v.taps, v.boundary, v.transform = int(self.taps), int(self.boundary), int(self.transform)
        return v


_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_sz = ctypes.c_size_t
_d = ctypes.c_double
_P = ctypes.POINTER(_Params)


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("prnu_default_params", _i, _P)
_sig("prnu_sda_groups", _i, _i64, _i64, ctypes.POINTER(_i64))
_sig("prnu_sda_average", _i, _vp, _i64, _i, _i, _i64, _vp, ctypes.POINTER(_i64), _vp)
_sig("prnu_rgb_to_luma", _i, _vp, _i64, _i, _i, _i, _i, _vp, _vp)
_sig("prnu_residual_workspace_bytes", _sz, _i, _i, _i, _P)
_sig("prnu_residual", _i, _vp, _i, _i, _i, _P, _i, _vp, _vp, _sz, _vp)
_sig("prnu_residual_u8", _i, _vp, _i, _i, _i, _P, _i, _vp, _vp, _sz, _vp)
_sig("prnu_fingerprint_accumulate", _i, _vp, _vp, _i, _i, _i, _vp, _vp, _vp)
_sig("prnu_finalize_workspace_bytes", _sz, _i, _i)
_sig("prnu_fingerprint_finalize", _i, _vp, _vp, _i, _i, _d, _i, _vp, _vp, _sz, _vp)
_sig("prnu_extract_workspace_bytes", _sz, _i, _i, _i, _i64, _P)
_sig("prnu_extract_fingerprint", _i, _vp, _i64, _i, _i, _i64, _P, _i, _d, _vp, _vp, _vp, ctypes.POINTER(_i64), _vp,
     _sz, _vp)
_sig("prnu_extract_fingerprint_stride", _i, _vp, _i64, _i, _i, _i64, _P, _i, _d, _vp, _vp, _vp, ctypes.POINTER(_i64),
     _vp, _sz, _vp)
_sig("prnu_extract_host_workspace_bytes", _sz, _i, _i, _i, _i64, _P)
_sig("prnu_extract_multi_host_workspace_bytes", _sz, _i64, _i, _i, _i, ctypes.POINTER(_i64), _i, _P)
_sig("prnu_extract_multi_host", _i, _vp, _i64, _i, _i, ctypes.POINTER(_i64), _i, _P, _i, _d, _vp, _vp,
     ctypes.POINTER(_i64), _vp, _sz, _vp)
_sig("prnu_extract_fingerprint_host", _i, _vp, _i64, _i, _i, _i64, _P, _i, _d, _vp, _vp, _vp,
     ctypes.POINTER(_i64), _vp, _sz, _vp)
_sig("prnu_ncc_workspace_bytes", _sz, _i, _i, _i)
_sig("prnu_ncc", _i, _vp, _vp, _i, _i, _i, _vp, _vp, _sz, _vp)
_sig("prnu_check_results", _i, _i, _vp, _i64, _vp)
_sig("prnu_pce_template", _i, _vp, _i, _vp, _i, _i, _i, _vp, _vp)
_sig("prnu_pce_plan_create", _i, _i, _i, _i, ctypes.POINTER(_sz), ctypes.POINTER(_vp))
_sig("prnu_pce", _i, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_pce_plan_destroy", _i, _vp)
_sig("prnu_pce_residual_spectrum", _i, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_pce_cached", _i, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_pce_cached_template", _i, _vp, _vp, _i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_wdft_plan_create", _i, _i, _i, _i, ctypes.POINTER(_sz), ctypes.POINTER(_vp))
_sig("prnu_wdft", _i, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_wdft_plan_destroy", _i, _vp)
_sig("prnu_block_plan_create", _i, _i, _i, _i, ctypes.POINTER(_i), ctypes.POINTER(_sz), ctypes.POINTER(_vp))
_sig("prnu_block_match", _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _sz, _vp)
_sig("prnu_block_plan_destroy", _i, _vp)
_VP = ctypes.POINTER(_Variant)
_sig("prnu_residual_variant_workspace_bytes", _sz, _i, _i, _i, _P, _VP)
_sig("prnu_residual_variant", _i, _vp, _i, _i, _i, _P, _VP, _i, _vp, _vp, _sz, _vp)
_sig("prnu_extract_variant_workspace_bytes", _sz, _i, _i, _i, _P, _VP)
_sig("prnu_extract_fingerprint_variant", _i, _vp, _i64, _i, _i, _i64, _P, _VP, _i, _d, _vp, _vp, _vp,
     ctypes.POINTER(_i64), _vp, _sz, _vp)
_sig("prnu_wavelet_filter", _i, _i, ctypes.POINTER(_d))
_sig("prnu_profile_begin", _i)
_sig("prnu_profile_end", _i, _i, ctypes.c_char_p, ctypes.POINTER(_d), ctypes.POINTER(_i64), ctypes.POINTER(_i))
_sig("prnu_last_error", ctypes.c_char_p)
_sig("prnu_kernel_launches", ctypes.c_uint64)
_sig("prnu_version", ctypes.c_char_p)


def _check(rc: int, where: str):
    if rc != 0:
        raise PrnuError(rc, where)


def _stream():
    """The current stream of the CURRENT device (every library call runs inside
    _on_device, which makes the tensors' device current)."""
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cuda_device(device) -> torch.device:
    """A concrete CUDA device (index filled in) for a device spec."""
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"expected a CUDA device, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def _on_device(fn):
    """Run a binding call with the device of its tensors (or of `self.device` for the
    plan/extractor classes) made current: the library launches on the current
    device's stream and keeps per-device state (kernel attributes, helper streams),
    so a call on cuda:N must run with cuda:N current.  All CUDA tensor arguments
    must live on that one device."""
    @functools.wraps(fn)
    def wrapped(*args, **kw):
        dev = None
        if args and isinstance(getattr(args[0], "device", None), torch.device) and not isinstance(args[0], torch.Tensor):
            dev = args[0].device
        for a in list(args) + list(kw.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                if dev is None:
                    dev = a.device
                elif a.device != dev:
                    raise ValueError(f"tensor on {a.device}, expected {dev} (one device per call)")
        if dev is None:
            return fn(*args, **kw)
        with torch.cuda.device(dev):
            return fn(*args, **kw)
    return wrapped


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, dtype, name: str, ndim=(2, 3)):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() not in ndim:
        raise ValueError(f"{name} must have {ndim} dims, got {t.dim()}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _params(p):
    return (p or DenoiseParams()).c()


def kernel_launches() -> int:
    """Kernels this library has launched so far (process-wide; cuFFT excluded)."""
    return int(_lib.prnu_kernel_launches())


def version() -> str:
    return _lib.prnu_version().decode()


# ---------------------------------------------------------------- a1
def sda_groups(m: int, depth: int) -> int:
    """floor(m/depth) SDA frames; DEPTH_EXCEEDS_FRAMES if depth > m."""
    n = _i64()
    _check(_lib.prnu_sda_groups(m, depth, ctypes.byref(n)), "prnu_sda_groups")
    return int(n.value)


@_on_device
def sda_average(frames: torch.Tensor, depth: int) -> torch.Tensor:
    """u8 [m,H,W] -> fp32 [floor(m/depth),H,W] SDA frames, bit-exact."""
    _dev(frames, torch.uint8, "frames", (3,))
    m, H, W = frames.shape
    ns = sda_groups(m, depth)
    out = torch.empty((ns, H, W), dtype=torch.float32, device=frames.device)
    _check(_lib.prnu_sda_average(_ptr(frames), m, H, W, depth, _ptr(out), None, _stream()), "prnu_sda_average")
    return out


prnu_sda_average = sda_average


# ---------------------------------------------------------------- f4 luma
@_on_device
def rgb_to_luma(rgb: torch.Tensor, layout: str = "planar", dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """u8 RGB -> luma [n,H,W] with the BT.601 weights (BASELINE config 3).

    layout "planar": rgb [n,3,H,W]; "interleaved": rgb [n,H,W,3].  dtype float32:
    RN_fp32((299R + 587G + 114B) / 1000); dtype uint8: the same rounded half to even."""
    _dev(rgb, torch.uint8, "rgb", (4,))
    if layout == "planar":
        n, c, H, W = rgb.shape
        lay = 0
    elif layout == "interleaved":
        n, H, W, c = rgb.shape
        lay = 1
    else:
        raise ValueError("layout must be 'planar' or 'interleaved'")
    if c != 3:
        raise ValueError("rgb must have 3 channels")
    if dtype not in (torch.float32, torch.uint8):
        raise ValueError("dtype must be float32 or uint8")
    out = torch.empty((n, H, W), dtype=dtype, device=rgb.device)
    _check(_lib.prnu_rgb_to_luma(_ptr(rgb), n, H, W, lay, 0 if dtype == torch.float32 else 1, _ptr(out), _stream()),
           "prnu_rgb_to_luma")
    return out


prnu_rgb_to_luma = rgb_to_luma


# ---------------------------------------------------------------- a2-a4
@_on_device
def residual(planes: torch.Tensor, params: DenoiseParams | None = None, zero_mean: bool = False,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """W = I - F(I) for fp32 or u8 planes [b,H,W] (or [H,W])."""
    squeeze = planes.dim() == 2
    if squeeze:
        planes = planes.unsqueeze(0)
    if planes.dtype not in (torch.float32, torch.uint8):
        raise TypeError("planes must be float32 or uint8")
    _dev(planes, planes.dtype, "planes", (3,))
    b, H, W = planes.shape
    p = _params(params)
    nbytes = _lib.prnu_residual_workspace_bytes(b, H, W, ctypes.byref(p))
    if nbytes == 0:   # invalid size/params: let the library name the error
        _check(_lib.prnu_residual(_ptr(planes), b, H, W, ctypes.byref(p), 0, _ptr(planes), _ptr(planes), 0, None),
               "prnu_residual")
    ws = _ws(nbytes, planes.device)
    if out is None:
        out = torch.empty((b, H, W), dtype=torch.float32, device=planes.device)
    fn = _lib.prnu_residual if planes.dtype == torch.float32 else _lib.prnu_residual_u8
    _check(fn(_ptr(planes), b, H, W, ctypes.byref(p), int(zero_mean), _ptr(out), _ptr(ws), nbytes, _stream()),
           "prnu_residual")
    return out[0] if squeeze else out


prnu_residual = residual


@_on_device
def residual_variant(planes: torch.Tensor, variant: DenoiseVariant, params: DenoiseParams | None = None,
                     zero_mean: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """f3: W = I - F(I) with a denoiser variant (db8 / pad + periodic / undecimated) for
    fp32 planes [b,H,W] (or [H,W]); same shrink and parameters as residual()."""
    squeeze = planes.dim() == 2
    if squeeze:
        planes = planes.unsqueeze(0)
    _dev(planes, torch.float32, "planes", (3,))
    b, H, W = planes.shape
    p = _params(params)
    v = variant.c()
    nbytes = _lib.prnu_residual_variant_workspace_bytes(b, H, W, ctypes.byref(p), ctypes.byref(v))
    if nbytes == 0:   # invalid size/params/variant: let the library name the error
        _check(_lib.prnu_residual_variant(_ptr(planes), b, H, W, ctypes.byref(p), ctypes.byref(v), 0,
                                          _ptr(planes), _ptr(planes), 0, None), "prnu_residual_variant")
    ws = _ws(nbytes, planes.device)
    if out is None:
        out = torch.empty((b, H, W), dtype=torch.float32, device=planes.device)
    _check(_lib.prnu_residual_variant(_ptr(planes), b, H, W, ctypes.byref(p), ctypes.byref(v), int(zero_mean),
                                      _ptr(out), _ptr(ws), nbytes, _stream()), "prnu_residual_variant")
    return out[0] if squeeze else out


prnu_residual_variant = residual_variant


def wavelet_filter(taps: int = 8) -> list:
    """The library's minimum-phase lowpass (the fp32 values its kernels use), host call."""
    h = (ctypes.c_double * taps)()
    _check(_lib.prnu_wavelet_filter(taps, h), "prnu_wavelet_filter")
    return list(h)


# ---------------------------------------------------------------- a5-a6
@_on_device
def fingerprint_accumulate(W: torch.Tensor, I: torch.Tensor, sum_WI: torch.Tensor, sum_I2: torch.Tensor):
    """sum_WI += W*I, sum_I2 += I^2 over the batch in order (Eq. 2)."""
    if W.dim() == 2:
        W, I = W.unsqueeze(0), I.unsqueeze(0)
    _dev(W, torch.float32, "W", (3,))
    _dev(I, torch.float32, "I", (3,))
    _dev(sum_WI, torch.float64, "sum_WI", (2,))
    _dev(sum_I2, torch.float64, "sum_I2", (2,))
    b, H, Wd = W.shape
    if I.shape != W.shape or sum_WI.shape != (H, Wd) or sum_I2.shape != (H, Wd):
        raise ValueError("dimension mismatch")
    _check(_lib.prnu_fingerprint_accumulate(_ptr(W), _ptr(I), b, H, Wd, _ptr(sum_WI), _ptr(sum_I2), _stream()),
           "prnu_fingerprint_accumulate")


prnu_fingerprint_accumulate = fingerprint_accumulate


@_on_device
def fingerprint_finalize(sum_WI: torch.Tensor, sum_I2: torch.Tensor, eps: float = 1e-6,
                         zero_mean: bool = True) -> torch.Tensor:
    """K = sum_WI / max(sum_I2, eps), then row/column zero-mean."""
    _dev(sum_WI, torch.float64, "sum_WI", (2,))
    _dev(sum_I2, torch.float64, "sum_I2", (2,))
    H, W = sum_WI.shape
    nbytes = _lib.prnu_finalize_workspace_bytes(H, W)
    ws = _ws(nbytes, sum_WI.device)
    K = torch.empty((H, W), dtype=torch.float32, device=sum_WI.device)
    _check(_lib.prnu_fingerprint_finalize(_ptr(sum_WI), _ptr(sum_I2), H, W, float(eps), int(zero_mean), _ptr(K),
                                          _ptr(ws), nbytes, _stream()), "prnu_fingerprint_finalize")
    return K


prnu_fingerprint_finalize = fingerprint_finalize


@dataclass
class Fingerprint:
    """A fingerprint and its MLE sums.  Fingerprints returned by Extractor /
    GraphExtractor ALIAS the extractor's own buffers (no allocation per call): the
    next call of the same extractor overwrites them — call .clone() to keep one."""
    K: torch.Tensor        # fp32 [H,W], zero-meaned K_hat
    sum_WI: torch.Tensor   # fp64 [H,W]
    sum_I2: torch.Tensor   # fp64 [H,W]
    n_sda: int             # denoise operations = floor(m/depth)
    depth: int
    frames: int

    def clone(self) -> "Fingerprint":
        return Fingerprint(self.K.clone(), self.sum_WI.clone(), self.sum_I2.clone(), self.n_sda, self.depth,
                           self.frames)


class Extractor:
    """Reusable fingerprint extractor for fixed (H, W, depth, batch): owns the
    workspace and accumulators so repeated calls allocate nothing.  The returned
    Fingerprint aliases those accumulators (see Fingerprint)."""

    def __init__(self, H: int, W: int, depth: int, batch: int = 16, params: DenoiseParams | None = None,
                 device="cuda", eps: float = 1e-6, host: bool = False):
        device = _cuda_device(device)
        self.device = device
        self.H, self.W, self.depth, self.batch, self.eps, self.host = H, W, depth, batch, eps, host
        self.p = _params(params)
        q = _lib.prnu_extract_host_workspace_bytes if host else _lib.prnu_extract_workspace_bytes
        self.nbytes = q(H, W, batch, depth, ctypes.byref(self.p))
        if self.nbytes == 0:
            raise PrnuError(4, "prnu_extract_workspace_bytes (invalid H/W/batch/depth/params)")
        self.ws = _ws(self.nbytes, device)
        self.sum_WI = torch.empty((H, W), dtype=torch.float64, device=device)
        self.sum_I2 = torch.empty((H, W), dtype=torch.float64, device=device)
        self.K = (torch.empty((H, W), dtype=torch.float32, pin_memory=True) if host
                  else torch.empty((H, W), dtype=torch.float32, device=device))

    @_on_device
    def __call__(self, frames: torch.Tensor) -> Fingerprint:
        if frames.dtype != torch.uint8 or frames.dim() != 3 or not frames.is_contiguous():
            raise TypeError("frames must be a contiguous uint8 [m,H,W] tensor")
        m, H, W = frames.shape
        if (H, W) != (self.H, self.W):
            raise ValueError("frame size differs from the extractor's")
        ns = _i64()
        if self.host:
            if frames.is_cuda:
                raise TypeError("host extractor takes CPU (pinned) frames")
            rc = _lib.prnu_extract_fingerprint_host(_ptr(frames), m, H, W, self.depth, ctypes.byref(self.p),
                                                    self.batch, self.eps, _ptr(self.K), _ptr(self.sum_WI),
                                                    _ptr(self.sum_I2), ctypes.byref(ns), _ptr(self.ws), self.nbytes,
                                                    _stream())
            _check(rc, "prnu_extract_fingerprint_host")
        else:
            _dev(frames, torch.uint8, "frames", (3,))
            rc = _lib.prnu_extract_fingerprint(_ptr(frames), m, H, W, self.depth, ctypes.byref(self.p), self.batch,
                                               self.eps, _ptr(self.K), _ptr(self.sum_WI), _ptr(self.sum_I2),
                                               ctypes.byref(ns), _ptr(self.ws), self.nbytes, _stream())
            _check(rc, "prnu_extract_fingerprint")
        return Fingerprint(self.K, self.sum_WI, self.sum_I2, int(ns.value), self.depth, m)


class GraphExtractor:
    """An Extractor whose whole call — SDA averaging, every level of every wave on the
    library's streams, the accumulation and the finalize — is captured once into a CUDA
    graph and replayed: one graph launch per fingerprint instead of ~10 kernel launches
    per wave (launch-bound small frames, e.g. BASELINE configs 1 and 4).  Frames are
    copied into a static device buffer of shape [m, H, W] (`self.frames`; write into it
    directly to skip the copy); results are bit-identical to Extractor's."""

    def __init__(self, m: int, H: int, W: int, depth: int, batch: int = 16, params: DenoiseParams | None = None,
                 device="cuda", eps: float = 1e-6):
        self.ex = Extractor(H, W, depth, batch, params, device, eps)
        self.device = self.ex.device
        self.frames = torch.empty((m, H, W), dtype=torch.uint8, device=self.device)
        self.graph = None
        self.n_sda = sda_groups(m, depth)

    @_on_device
    def __call__(self, frames: torch.Tensor | None = None) -> Fingerprint:
        if frames is not None and frames.data_ptr() != self.frames.data_ptr():
            self.frames.copy_(frames)
        if self.graph is None:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):   # warm-up outside capture: kernel attributes, stream pool
                self.ex(self.frames)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.ex(self.frames)
        self.graph.replay()
        ex = self.ex
        return Fingerprint(ex.K, ex.sum_WI, ex.sum_I2, self.n_sda, ex.depth, self.frames.shape[0])


class CameraBatchExtractor:
    """Fingerprints of many independent videos (cameras) of the same size and depth:
    one Extractor (workspace, accumulators) per stream, cameras dealt round-robin over
    `streams` CUDA streams so small per-camera waves overlap on the GPU (BASELINE
    config 4: 64 cameras x 300 frames 1280x720 at depth 30)."""

    def __init__(self, H: int, W: int, depth: int, batch: int = 16, streams: int = 8,
                 params: DenoiseParams | None = None, device="cuda", eps: float = 1e-6):
        self.H, self.W = H, W
        device = _cuda_device(device)
        self.exs = [Extractor(H, W, depth, batch, params, device, eps) for _ in range(streams)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(streams)]
        self.device = device

    @_on_device
    def __call__(self, videos) -> torch.Tensor:
        """videos: a sequence of uint8 [m, H, W] device tensors (or a [n, m, H, W] tensor);
        returns K fp32 [n, H, W]."""
        n = len(videos)
        K = torch.empty((n, self.H, self.W), dtype=torch.float32, device=self.device)
        cur = torch.cuda.current_stream()
        for s_ in self.streams:
            s_.wait_stream(cur)
        for c in range(n):
            j = c % len(self.streams)
            with torch.cuda.stream(self.streams[j]):
                K[c].copy_(self.exs[j](videos[c]).K)
        for s_ in self.streams:
            cur.wait_stream(s_)
        return K


class MultiExtractor:
    """Fingerprints at several SDA depths from ONE upload of a host (pinned) frame
    stack [m][H][W]; owns the device workspace (which holds the whole stack)."""

    def __init__(self, m: int, H: int, W: int, depths, batch: int = 64, params: DenoiseParams | None = None,
                 device="cuda", eps: float = 1e-6):
        self.m, self.H, self.W, self.batch, self.eps = m, H, W, batch, eps
        device = _cuda_device(device)
        self.device = device
        self.depths = [int(d) for d in depths]
        self.p = _params(params)
        self._d = (_i64 * len(self.depths))(*self.depths)
        self.nbytes = _lib.prnu_extract_multi_host_workspace_bytes(m, H, W, batch, self._d, len(self.depths),
                                                                   ctypes.byref(self.p))
        if self.nbytes == 0:
            raise PrnuError(4, "prnu_extract_multi_host_workspace_bytes (invalid m/H/W/batch/depths/params)")
        self.ws = _ws(self.nbytes, device)
        self.sums = torch.empty((len(self.depths), 2, H, W), dtype=torch.float64, device=device)
        self.K = torch.empty((len(self.depths), H, W), dtype=torch.float32, pin_memory=True)
        self.n_sda = [0] * len(self.depths)

    @_on_device
    def __call__(self, frames_host: torch.Tensor) -> torch.Tensor:
        if frames_host.is_cuda or frames_host.dtype != torch.uint8 or not frames_host.is_contiguous():
            raise TypeError("frames must be a contiguous uint8 CPU (pinned) tensor")
        if tuple(frames_host.shape) != (self.m, self.H, self.W):
            raise ValueError("frame stack shape differs from the extractor's")
        ns = (_i64 * len(self.depths))()
        _check(_lib.prnu_extract_multi_host(_ptr(frames_host), self.m, self.H, self.W, self._d, len(self.depths),
                                            ctypes.byref(self.p), self.batch, self.eps, _ptr(self.K),
                                            _ptr(self.sums), ns, _ptr(self.ws), self.nbytes, _stream()),
               "prnu_extract_multi_host")
        self.n_sda = list(ns)
        return self.K


@_on_device
def extract_fingerprint(frames: torch.Tensor, depth: int, params: DenoiseParams | None = None, batch: int = 16,
                        eps: float = 1e-6) -> Fingerprint:
    """The three steps of P:58-60 (average, denoise, MLE) + finalize, on device frames."""
    m, H, W = frames.shape
    sda_groups(m, depth)
    return Extractor(H, W, depth, batch, params, frames.device, eps)(frames)


prnu_extract_fingerprint = extract_fingerprint


@_on_device
def extract_fingerprint_stride(frames: torch.Tensor, stride: int, params: DenoiseParams | None = None,
                               batch: int = 16, eps: float = 1e-6) -> Fingerprint:
    """f4 I-frame emulation: conventional fingerprint of the
    frames 0, stride, 2 stride, ... (n = ceil(m / stride) denoisings)."""
    _dev(frames, torch.uint8, "frames", (3,))
    m, H, W = frames.shape
    p = _params(params)
    nbytes = _lib.prnu_extract_workspace_bytes(H, W, batch, 1, ctypes.byref(p))
    ws = _ws(nbytes, frames.device)
    s_wi = torch.empty((H, W), dtype=torch.float64, device=frames.device)
    s_i2 = torch.empty_like(s_wi)
    K = torch.empty((H, W), dtype=torch.float32, device=frames.device)
    n = _i64()
    _check(_lib.prnu_extract_fingerprint_stride(_ptr(frames), m, H, W, stride, ctypes.byref(p), batch, eps, _ptr(K),
                                                _ptr(s_wi), _ptr(s_i2), ctypes.byref(n), _ptr(ws), nbytes, _stream()),
           "prnu_extract_fingerprint_stride")
    return Fingerprint(K, s_wi, s_i2, int(n.value), 1, m)


prnu_extract_fingerprint_stride = extract_fingerprint_stride


@_on_device
def extract_fingerprint_variant(frames: torch.Tensor, depth: int, variant: DenoiseVariant,
                                params: DenoiseParams | None = None, batch: int = 16,
                                eps: float = 1e-6) -> Fingerprint:
    """f3: the fingerprint pipeline (SDA average, denoise, MLE, finalize) with a
    denoiser variant (prnu_extract_fingerprint_variant: waves of `batch` SDA frames
    through the variant passes, accumulated in ascending group order)."""
    _dev(frames, torch.uint8, "frames", (3,))
    m, H, W = frames.shape
    p = _params(params)
    v = variant.c()
    nbytes = _lib.prnu_extract_variant_workspace_bytes(H, W, batch, ctypes.byref(p), ctypes.byref(v))
    if nbytes == 0:
        raise PrnuError(4, "invalid arguments for the variant extraction")
    ws = _ws(nbytes, frames.device)
    s_wi = torch.empty((H, W), dtype=torch.float64, device=frames.device)
    s_i2 = torch.empty_like(s_wi)
    K = torch.empty((H, W), dtype=torch.float32, device=frames.device)
    n = _i64()
    _check(_lib.prnu_extract_fingerprint_variant(_ptr(frames), m, H, W, depth, ctypes.byref(p), ctypes.byref(v),
                                                 batch, eps, _ptr(K), _ptr(s_wi), _ptr(s_i2), ctypes.byref(n),
                                                 _ptr(ws), nbytes, _stream()), "prnu_extract_fingerprint_variant")
    return Fingerprint(K, s_wi, s_i2, int(n.value), depth, m)


prnu_extract_fingerprint_variant = extract_fingerprint_variant


# ---------------------------------------------------------------- a7-a8
CHECK_NCC, CHECK_PCE, CHECK_SUM_I2 = 0, 1, 2


@_on_device
def check_results(kind: int, values: torch.Tensor) -> None:
    """prnu_check_results: raise PrnuError 7 (ConstantInput) for NaN NCC values,
    8 (DegenerateSurface) for a zero PCE peak (the surface is constant), 6
    (EmptyAccumulator) for an all-zero sum_I2.  Synchronous (waits for the current
    stream)."""
    _dev(values, torch.float64, "values", (1, 2, 3))
    _check(_lib.prnu_check_results(int(kind), _ptr(values), values.numel(), _stream()), "prnu_check_results")


@_on_device
def ncc(a: torch.Tensor, b: torch.Tensor, check: bool = False) -> torch.Tensor:
    """Aligned Pearson correlation per plane (R-16), fp64 [batch] (or 0-dim).  A constant
    operand gives NaN in-band; check=True raises PrnuError 7 instead (synchronous)."""
    squeeze = a.dim() == 2
    if squeeze:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    _dev(a, torch.float32, "a", (3,))
    _dev(b, torch.float32, "b", (3,))
    if a.shape != b.shape:
        raise ValueError("dimension mismatch")
    n, H, W = a.shape
    nbytes = _lib.prnu_ncc_workspace_bytes(n, H, W)
    ws = _ws(nbytes, a.device)
    out = torch.empty((n,), dtype=torch.float64, device=a.device)
    _check(_lib.prnu_ncc(_ptr(a), _ptr(b), n, H, W, _ptr(out), _ptr(ws), nbytes, _stream()), "prnu_ncc")
    if check:
        check_results(CHECK_NCC, out)
    return out[0] if squeeze else out


prnu_ncc = ncc


@_on_device
def pce_template(K: torch.Tensor, Iq: torch.Tensor) -> torch.Tensor:
    """T = K (.) Iq (R-18); K fp32 [H,W] or [b,H,W], Iq u8 [b,H,W] or [H,W]."""
    if Iq.dim() == 2:
        Iq = Iq.unsqueeze(0)
    Kb = K.unsqueeze(0) if K.dim() == 2 else K
    _dev(Kb, torch.float32, "K", (3,))
    _dev(Iq, torch.uint8, "Iq", (3,))
    b, H, W = Iq.shape
    T = torch.empty((b, H, W), dtype=torch.float32, device=Iq.device)
    _check(_lib.prnu_pce_template(_ptr(Kb), Kb.shape[0], _ptr(Iq), b, H, W, _ptr(T), _stream()),
           "prnu_pce_template")
    return T


@dataclass
class PceResult:
    pce: torch.Tensor     # fp64 [b]
    peak_y: torch.Tensor  # int32 [b]
    peak_x: torch.Tensor  # int32 [b]
    peak: torch.Tensor    # fp64 [b]

    def decision(self) -> torch.Tensor:
        return self.pce > PCE_THRESHOLD   # strict


class PcePlan:
    """PCE plan (the library's row / column FFT kernels, or cuFFT where a size has no
    radix plan) + workspace for [batch][H][W] residual/template pairs."""

    def __init__(self, H: int, W: int, batch: int = 1, device="cuda"):
        self.H, self.W, self.batch = H, W, batch
        device = _cuda_device(device)
        self.device = device
        nb = _sz()
        h = _vp()
        with torch.cuda.device(device):   # the cuFFT plans belong to the current device
            _check(_lib.prnu_pce_plan_create(H, W, batch, ctypes.byref(nb), ctypes.byref(h)), "prnu_pce_plan_create")
        self._h = h
        self.nbytes = int(nb.value)
        self.ws = _ws(self.nbytes, device)
        self.out = PceResult(torch.empty(batch, dtype=torch.float64, device=device),
                             torch.empty(batch, dtype=torch.int32, device=device),
                             torch.empty(batch, dtype=torch.int32, device=device),
                             torch.empty(batch, dtype=torch.float64, device=device))

    @_on_device
    def __call__(self, R: torch.Tensor, T: torch.Tensor, exclusion_half: int = 5, aligned: bool = False) -> PceResult:
        if R.dim() == 2:
            R, T = R.unsqueeze(0), T.unsqueeze(0)
        _dev(R, torch.float32, "residual", (3,))
        _dev(T, torch.float32, "template", (3,))
        if R.shape != (self.batch, self.H, self.W) or T.shape != R.shape:
            raise ValueError("dimension mismatch with the plan")
        o = self.out
        _check(_lib.prnu_pce(self._h, _ptr(R), _ptr(T), self.batch, exclusion_half, int(aligned), _ptr(o.pce),
                             _ptr(o.peak_y), _ptr(o.peak_x), _ptr(o.peak), _ptr(self.ws), self.nbytes, _stream()),
               "prnu_pce")
        return PceResult(o.pce.clone(), o.peak_y.clone(), o.peak_x.clone(), o.peak.clone())

    @_on_device
    def set_residual(self, R: torch.Tensor):
        """Cache FFT2 of the residual batch in the plan's workspace (prnu_pce_residual_spectrum)."""
        if R.dim() == 2:
            R = R.unsqueeze(0)
        _dev(R, torch.float32, "residual", (3,))
        if R.shape != (self.batch, self.H, self.W):
            raise ValueError("dimension mismatch with the plan")
        _check(_lib.prnu_pce_residual_spectrum(self._h, _ptr(R), _ptr(self.ws), self.nbytes, _stream()),
               "prnu_pce_residual_spectrum")

    @_on_device
    def match(self, T: torch.Tensor, exclusion_half: int = 5, aligned: bool = False) -> PceResult:
        """PCE of the cached residuals (set_residual) against templates T (prnu_pce_cached)."""
        if T.dim() == 2:
            T = T.unsqueeze(0)
        _dev(T, torch.float32, "template", (3,))
        if T.shape != (self.batch, self.H, self.W):
            raise ValueError("dimension mismatch with the plan")
        o = self.out
        _check(_lib.prnu_pce_cached(self._h, _ptr(T), self.batch, exclusion_half, int(aligned), _ptr(o.pce),
                                    _ptr(o.peak_y), _ptr(o.peak_x), _ptr(o.peak), _ptr(self.ws), self.nbytes,
                                    _stream()), "prnu_pce_cached")
        return PceResult(o.pce.clone(), o.peak_y.clone(), o.peak_x.clone(), o.peak.clone())

    @_on_device
    def match_template(self, K: torch.Tensor, Iq: torch.Tensor, exclusion_half: int = 5,
                       aligned: bool = False) -> PceResult:
        """PCE of the cached residuals against the templates K (.) Iq (prnu_pce_cached_template):
        the same result as match(pce_template(K, Iq)) without materialising the templates."""
        Kb = K.unsqueeze(0) if K.dim() == 2 else K
        if Iq.dim() == 2:
            Iq = Iq.unsqueeze(0)
        _dev(Kb, torch.float32, "K", (3,))
        _dev(Iq, torch.uint8, "Iq", (3,))
        if Iq.shape != (self.batch, self.H, self.W) or Kb.shape[1:] != (self.H, self.W):
            raise ValueError("dimension mismatch with the plan")
        o = self.out
        _check(_lib.prnu_pce_cached_template(self._h, _ptr(Kb), Kb.shape[0], _ptr(Iq), self.batch, exclusion_half,
                                             int(aligned), _ptr(o.pce), _ptr(o.peak_y), _ptr(o.peak_x),
                                             _ptr(o.peak), _ptr(self.ws), self.nbytes, _stream()),
               "prnu_pce_cached_template")
        return PceResult(o.pce.clone(), o.peak_y.clone(), o.peak_x.clone(), o.peak.clone())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            with torch.cuda.device(self.device):
                _lib.prnu_pce_plan_destroy(h)
            self._h = None


class PceMatrix:
    """Camera identification (BASELINE config 4): the PCE of `batch` query residuals
    against the templates K_c (.) Iq of many fingerprints K_c.  One PcePlan per stream,
    each holding the cached query-residual spectrum; fingerprints are dealt
    round-robin over the streams so consecutive fingerprints' kernels overlap."""

    def __init__(self, H: int, W: int, batch: int, streams: int = 4, device="cuda"):
        device = _cuda_device(device)
        self.H, self.W, self.batch, self.device = H, W, batch, device
        self.plans = [PcePlan(H, W, batch, device) for _ in range(streams)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(streams)]
        self.Iq = None

    @_on_device
    def set_queries(self, R: torch.Tensor, Iq: torch.Tensor):
        """R: zero-mean query residuals fp32 [batch][H][W]; Iq: the query frames u8."""
        for p in self.plans:
            p.set_residual(R)
        self.Iq = Iq

    @_on_device
    def __call__(self, Ks, exclusion_half: int = 5) -> PceResult:
        """Ks: a sequence of fp32 [H][W] fingerprints (or [n][H][W]); returns PceResult
        fields of shape [n][batch] (row c: fingerprint c against every query)."""
        if self.Iq is None:
            raise RuntimeError("set_queries first")
        cur = torch.cuda.current_stream()
        for s_ in self.streams:
            s_.wait_stream(cur)
        res = []
        for c in range(len(Ks)):
            j = c % len(self.plans)
            with torch.cuda.stream(self.streams[j]):
                res.append(self.plans[j].match_template(Ks[c], self.Iq, exclusion_half))
        for s_ in self.streams:
            cur.wait_stream(s_)
        return PceResult(torch.stack([r.pce for r in res]), torch.stack([r.peak_y for r in res]),
                         torch.stack([r.peak_x for r in res]), torch.stack([r.peak for r in res]))


class WdftPlan:
    """f2: Wiener filtering of [batch][H][W] zero-mean fingerprints in the DFT domain
    (S:151 option; R-23): K' = IDFT2(F * s2 / max(m, s2)) with F = DFT2(K),
    s2 = mean(K^2), m = min over windows 3..9 of the box mean of |F|^2 / (HW)."""

    def __init__(self, H: int, W: int, batch: int = 1, device="cuda"):
        self.H, self.W, self.batch = H, W, batch
        device = _cuda_device(device)
        self.device = device
        nb = _sz()
        h = _vp()
        with torch.cuda.device(device):
            _check(_lib.prnu_wdft_plan_create(H, W, batch, ctypes.byref(nb), ctypes.byref(h)), "prnu_wdft_plan_create")
        self._h = h
        self.nbytes = int(nb.value)
        self.ws = _ws(self.nbytes, device)

    @_on_device
    def __call__(self, K: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        squeeze = K.dim() == 2
        if squeeze:
            K = K.unsqueeze(0)
        _dev(K, torch.float32, "K", (3,))
        if K.shape != (self.batch, self.H, self.W):
            raise ValueError("dimension mismatch with the plan")
        out = torch.empty_like(K) if out is None else out
        _check(_lib.prnu_wdft(self._h, _ptr(K), _ptr(out), _ptr(self.ws), self.nbytes, _stream()), "prnu_wdft")
        return out[0] if squeeze else out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            with torch.cuda.device(self.device):
                _lib.prnu_wdft_plan_destroy(h)
            self._h = None


@_on_device
def wdft(K: torch.Tensor) -> torch.Tensor:
    b = 1 if K.dim() == 2 else K.shape[0]
    return WdftPlan(K.shape[-2], K.shape[-1], b, K.device)(K)


prnu_wdft = wdft


@_on_device
def pce(R: torch.Tensor, T: torch.Tensor, exclusion_half: int = 5, aligned: bool = False,
        check: bool = False) -> PceResult:
    """PCE per pair (prnu_pce).  A degenerate (constant) surface is reported in-band (peak 0,
    PCE at the cap); check=True raises PrnuError 8 instead (synchronous)."""
    b = 1 if R.dim() == 2 else R.shape[0]
    res = PcePlan(R.shape[-2], R.shape[-1], b, R.device)(R, T, exclusion_half, aligned)
    if check:
        check_results(CHECK_PCE, res.peak.reshape(-1))
    return res


prnu_pce = pce


# ---------------------------------------------------------------- f4: H0/H1 detection rates (host logic)
PCE_THRESHOLD = 60.0   # P:259 "PCE higher than 60" -> match; strict (R-20)


def detection_rates(pce_matrix, threshold: float = PCE_THRESHOLD) -> dict:
    """Camera-identification decisions from a square PCE matrix M[q, c] (query q
    against fingerprint c; the diagonal are the H1 pairs, the rest H0): TPR =
    share of H1 pairs with PCE > threshold, FPR = share of H0 pairs with
    PCE > threshold (strict, R-20).  Host-side bookkeeping over device results."""
    import numpy as np
    M = np.asarray(pce_matrix, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("pce_matrix must be square [queries, fingerprints]")
    eye = np.eye(M.shape[0], dtype=bool)
    h1, h0 = M[eye], M[~eye]
    return {"tpr": float(np.mean(h1 > threshold)), "fpr": float(np.mean(h0 > threshold)) if h0.size else 0.0,
            "n_h1": int(h1.size), "n_h0": int(h0.size)}


def roc(pce_h1, pce_h0):
    """ROC of the PCE detector: thresholds at every observed score (descending),
    returns (fpr, tpr, auc) with the decision PCE > threshold; AUC by the
    trapezoid rule from (0, 0) to (1, 1)."""
    import numpy as np
    h1 = np.asarray(pce_h1, dtype=np.float64).ravel()
    h0 = np.asarray(pce_h0, dtype=np.float64).ravel()
    if h1.size == 0 or h0.size == 0:
        raise ValueError("need H1 and H0 scores")
    th = np.unique(np.concatenate([h1, h0]))[::-1]
    tpr = np.array([0.0] + [float(np.mean(h1 >= t)) for t in th])
    fpr = np.array([0.0] + [float(np.mean(h0 >= t)) for t in th])
    auc = float(np.sum((fpr[1:] - fpr[:-1]) * (tpr[1:] + tpr[:-1]) / 2.0))
    return fpr, tpr, auc


class BlockPlan:
    """f1 block-wise matching: per-tile aligned PCE and
    NCC over block x block tiles (edge tiles kept), row-major tile order."""

    def __init__(self, H: int, W: int, block: int = 500, device="cuda"):
        self.H, self.W, self.block = H, W, block
        device = _cuda_device(device)
        n = _i()
        nb = _sz()
        h = _vp()
        with torch.cuda.device(device):
            _check(_lib.prnu_block_plan_create(H, W, block, ctypes.byref(n), ctypes.byref(nb), ctypes.byref(h)),
                   "prnu_block_plan_create")
        self._h = h
        self.n_tiles = int(n.value)
        self.nbytes = int(nb.value)
        self.ws = _ws(self.nbytes, device)
        self.device = device

    def tiles(self):
        """[(y, x, h, w)] in row-major order."""
        b = self.block
        return [(y, x, min(b, self.H - y), min(b, self.W - x)) for y in range(0, self.H, b)
                for x in range(0, self.W, b)]

    @_on_device
    def __call__(self, R: torch.Tensor, T: torch.Tensor, exclusion_half: int = 5):
        _dev(R, torch.float32, "residual", (2,))
        _dev(T, torch.float32, "template", (2,))
        if R.shape != (self.H, self.W) or T.shape != R.shape:
            raise ValueError("dimension mismatch with the plan")
        pce = torch.empty(self.n_tiles, dtype=torch.float64, device=R.device)
        ncc = torch.empty(self.n_tiles, dtype=torch.float64, device=R.device)
        _check(_lib.prnu_block_match(self._h, _ptr(R), _ptr(T), exclusion_half, _ptr(pce), _ptr(ncc), _ptr(self.ws),
                                     self.nbytes, _stream()), "prnu_block_match")
        return pce, ncc

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            with torch.cuda.device(self.device):
                _lib.prnu_block_plan_destroy(h)
            self._h = None


@_on_device
def block_match(R: torch.Tensor, T: torch.Tensor, block: int = 500, exclusion_half: int = 5):
    return BlockPlan(R.shape[-2], R.shape[-1], block, R.device)(R, T, exclusion_half)


prnu_block_match = block_match


def header_symbols() -> list[str]:
    """Every function declared in include/prnu.h."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(prnu_[a-z0-9_]+)\s*\(", txt)))
