"""Python binding of libconv.so (include/conv.h) -- argument marshalling only.

Every step of a convolution runs in the library's sm_100a kernels; this module
passes tensor pointers, sizes and the caller's CUDA stream through ctypes.
PyTorch is used only for device memory and streams.  There is no CPU
fallback: if ``libconv.so`` is missing or no sm_100 device is present the
calls raise.
"""
from __future__ import annotations

import ctypes
import json
import os
import threading
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# CONV_LIB: an A/B build of the same sources with study flags
# (scripts/build_ab.py, e.g. _ab_ffma2/libconv.so); experiments only
LIB_PATH = os.environ.get("CONV_LIB") or os.path.join(_HERE, "libconv.so")

CONV_OK = 0
CONV_ERR_INVALID_ARGUMENT = 1
CONV_ERR_INFEASIBLE = 2
CONV_ERR_CUDA = 3
CONV_ERR_UNSUPPORTED_DEVICE = 4

PATHS = {"auto": 0, "fp32_simt": 1, "tf32": 2, "bf16": 3, "fp32_tc": 4}
PATH_NAMES = {v: k for k, v in PATHS.items()}

# Every symbol include/conv.h declares (tests check the library exports them).
EXPORTED = (
    "conv_plan_create", "conv_plan_create_offline", "conv_plan_create_strided", "conv_plan_create_strided_offline",
    "conv_plan_create_dilated", "conv_plan_create_dilated_offline",
    "conv_plan_create_padded", "conv_plan_create_padded_offline",
    "conv_plan_set_path", "conv_plan_set_tile", "conv_plan_workspace_bytes",
    "conv_plan_num_kernels", "conv_plan_path", "conv_plan_describe", "conv_plan_destroy",
    "conv_run", "conv_run_events", "conv_plan_host_run_bytes", "conv_run_host",
    "conv_last_error", "conv_last_status", "conv_version", "conv_model_dv", "conv_model_dv_matmul",
    "conv_model_footprint",
)


class ConvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[conv status {status}] {msg}")
        self.status = status


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libconv.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        vp, sz, i, d = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double
        sig = {
            "conv_plan_create": (vp, [i] * 7),
            "conv_plan_create_offline": (vp, [i] * 8 + [sz, sz]),
            "conv_plan_create_strided": (vp, [i] * 8),
            "conv_plan_create_strided_offline": (vp, [i] * 9 + [sz, sz]),
            "conv_plan_create_dilated": (vp, [i] * 9),
            "conv_plan_create_dilated_offline": (vp, [i] * 10 + [sz, sz]),
            "conv_plan_create_padded": (vp, [i] * 11),
            "conv_plan_create_padded_offline": (vp, [i] * 12 + [sz, sz]),
            "conv_plan_set_path": (i, [vp, i]),
            "conv_plan_set_tile": (i, [vp, ctypes.c_char_p]),
            "conv_plan_workspace_bytes": (sz, [vp]),
            "conv_plan_num_kernels": (i, [vp]),
            "conv_plan_path": (i, [vp]),
            "conv_plan_describe": (i, [vp, ctypes.c_char_p, sz]),
            "conv_plan_destroy": (None, [vp]),
            "conv_run": (i, [vp, vp, vp, vp, vp, vp]),
            "conv_run_events": (i, [vp, vp, vp, vp, vp, vp, ctypes.POINTER(vp), i]),
            "conv_plan_host_run_bytes": (sz, [vp]),
            "conv_run_host": (i, [vp, vp, vp, vp, vp, vp]),
            "conv_last_error": (ctypes.c_char_p, []),
            "conv_last_status": (ctypes.c_int, []),
            "conv_version": (ctypes.c_char_p, []),
            "conv_model_dv": (d, [ctypes.POINTER(i), ctypes.POINTER(d), ctypes.POINTER(d), ctypes.POINTER(d)]),
            "conv_model_dv_matmul": (d, [ctypes.POINTER(i), ctypes.POINTER(d), ctypes.POINTER(d)]),
            "conv_model_footprint": (d, [ctypes.POINTER(d)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load_library().conv_last_error().decode()


def version() -> str:
    return load_library().conv_version().decode()


def _check(status: int):
    if status != CONV_OK:
        raise ConvError(status, last_error())


def torch_current_stream(device=None):
    import torch
    return torch.cuda.current_stream(device)


def _stream_handle(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class ConvPlan:
    """A plan for Eq. 1 with OUTPUT extents H x W; with
    ``stride`` U > 1, ``dilation`` D > 1, ``padding`` (ph, pw) (or explicit
    ``in_hw``) the general form Out[n,k,h,w] = sum In[n,c,U*h+D*r-ph,U*w+D*s-pw]
    Ker[k,c,r,s], In zero outside the input (conv_plan_create_padded)."""

    def __init__(self, N: int, K: int, C: int, H: int, W: int, R: int, S: int,
                 path: str = "auto", tile: Optional[str] = None, offline_device: Optional[dict] = None,
                 stride: int = 1, in_hw: Optional[tuple] = None, dilation: int = 1, padding=0):
        """``offline_device`` = dict(sms=, smem_optin=, l2_bytes=) plans for a
        described device without touching CUDA (describe-only plan).
        ``in_hw`` = (Hin, Win) input extents of a strided plan (default the
        minimal ((H-1)*U+D*(R-1)+1-2ph, (W-1)*U+D*(S-1)+1-2pw)); H, W must
        equal the floor output extents (Hin+2ph-D*(R-1)-1)//U+1, likewise W.
        ``padding`` is an int or (ph, pw)."""
        lib = load_library()
        self._lib = lib
        ph, pw = (padding, padding) if isinstance(padding, int) else tuple(padding)
        strided = stride != 1 or dilation != 1 or ph != 0 or pw != 0 or in_hw is not None
        Re, Se = dilation * (R - 1) + 1, dilation * (S - 1) + 1     # dilated kernel extents
        if strided:
            Hin, Win = in_hw if in_hw is not None else ((H - 1) * stride + Re - 2 * ph, (W - 1) * stride + Se - 2 * pw)
            if (stride >= 1 and dilation >= 1 and Hin + 2 * ph >= Re and Win + 2 * pw >= Se
                    and ((Hin + 2 * ph - Re) // stride + 1, (Win + 2 * pw - Se) // stride + 1) != (H, W)):
                raise ValueError(f"output {H}x{W} does not match input {Hin}x{Win}, kernel {R}x{S}, "
                                 f"stride {stride}, dilation {dilation}, padding {(ph, pw)}")
        else:
            Hin, Win = H + R - 1, W + S - 1
        self.shape = (N, K, C, H, W, R, S)
        self.stride = stride
        self.dilation = dilation
        self.padding = (ph, pw)
        self.in_hw = (Hin, Win)
        if offline_device is not None:
            d = offline_device
            dev = (int(d["sms"]), int(d["smem_optin"]), int(d["l2_bytes"]))
            h = (lib.conv_plan_create_padded_offline(N, K, C, Hin, Win, R, S, stride, dilation, ph, pw, *dev) if strided
                 else lib.conv_plan_create_offline(N, K, C, H, W, R, S, *dev))
        else:
            h = (lib.conv_plan_create_padded(N, K, C, Hin, Win, R, S, stride, dilation, ph, pw) if strided
                 else lib.conv_plan_create(N, K, C, H, W, R, S))
        if not h:
            raise ConvError(lib.conv_last_status(), last_error())
        self._h = ctypes.c_void_p(h)
        # the device the library bound the plan to (the current one); runs
        # must pass tensors on it (checked in run / run_events)
        self.device_index = None
        if offline_device is None:
            import torch
            self.device_index = torch.cuda.current_device()
        self._shapes_cache = tuple(self._shapes_sizes())
        if path != "auto":
            self.set_path(path)
        if tile:
            self.set_tile(tile)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.conv_plan_destroy(h)
            self._h = None

    def set_path(self, path: str):
        if path not in PATHS:
            raise ValueError(f"unknown path {path!r}")
        _check(self._lib.conv_plan_set_path(self._h, PATHS[path]))

    def set_tile(self, spec: Optional[str]):
        _check(self._lib.conv_plan_set_tile(self._h, (spec or "").encode()))

    @property
    def path(self) -> str:
        return PATH_NAMES[self._lib.conv_plan_path(self._h)]

    @property
    def workspace_bytes(self) -> int:
        return int(self._lib.conv_plan_workspace_bytes(self._h))

    @property
    def num_kernels(self) -> int:
        return int(self._lib.conv_plan_num_kernels(self._h))

    @property
    def host_run_bytes(self) -> int:
        return int(self._lib.conv_plan_host_run_bytes(self._h))

    def describe(self) -> dict:
        n = self._lib.conv_plan_describe(self._h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        self._lib.conv_plan_describe(self._h, buf, n + 1)
        return json.loads(buf.value.decode())

    # -- execution -----------------------------------------------------------
    def _shapes(self):
        N, K, C, H, W, R, S = self.shape
        return (N, C) + tuple(self.in_hw), (K, C, R, S), (N, K, H, W)

    def _shapes_sizes(self):
        import torch
        return [torch.Size(s) for s in self._shapes()]

    def _check_tensors(self, inp, ker, out):
        si, sk, so = self._shapes_cache
        for t, s, name in ((inp, si, "in"), (ker, sk, "ker"), (out, so, "out")):
            if not (t.is_cuda and t.dtype is _f32() and t.shape == s and t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float32 CUDA tensor of shape {tuple(s)}, "
                                 f"got {t.dtype} {tuple(t.shape)} on {t.device}")
            if t.device.index != self.device_index:
                raise ValueError(f"{name} is on {t.device} but the plan was created on cuda:{self.device_index}")

    def new_workspace(self, device=None):
        import torch
        n = self.workspace_bytes
        return torch.empty(max(n, 1), dtype=torch.uint8, device=device or "cuda")

    def new_output(self, device=None):
        import torch
        return torch.empty(self._shapes()[2], dtype=torch.float32, device=device or "cuda")

    def run(self, inp, ker, out=None, workspace=None, stream=None):
        """Out = Eq. 1 (In, Ker), asynchronous on ``stream`` (default: torch's
        current stream).  Returns ``out``.  Buffers this call allocates (out,
        workspace) are allocated on ``stream`` (torch's caching allocator
        then never hands them to other work while the kernels run)."""
        import torch
        with torch.cuda.device(inp.device):
            alloc = torch.cuda.stream(stream) if stream is not None else _nullcontext()
            with alloc:
                if out is None:
                    out = self.new_output(inp.device)
                if workspace is None and self.workspace_bytes:
                    workspace = self.new_workspace(inp.device)
            self._check_tensors(inp, ker, out)
            ws = workspace.data_ptr() if workspace is not None and self.workspace_bytes else None
            _check(self._lib.conv_run(self._h, inp.data_ptr(), ker.data_ptr(), out.data_ptr(), ws,
                                      _stream_handle(stream)))
        return out

    def run_events(self, inp, ker, out, workspace, events: Sequence, stream=None):
        """conv_run recording ``events`` (torch.cuda.Event, enable_timing) around
        each kernel on ``stream``."""
        self._check_tensors(inp, ker, out)
        n = len(events)
        s = stream if stream is not None else torch_current_stream(inp.device)
        for e in events:
            if not e.cuda_event:          # torch creates the cudaEvent_t lazily, on first record
                e.record(s)
        arr = (ctypes.c_void_p * n)(*[e.cuda_event for e in events])
        ws = workspace.data_ptr() if workspace is not None and self.workspace_bytes else None
        _check(self._lib.conv_run_events(self._h, inp.data_ptr(), ker.data_ptr(), out.data_ptr(), ws,
                                         _stream_handle(stream), arr, n))

    def run_host(self, in_host, ker_host, out_host, device_buffer, stream=None):
        """End-to-end call with (pinned) host tensors: H2D, conv, D2H on one
        stream inside the library.  Asynchronous."""
        import torch
        si, sk, so = self._shapes()
        for t, s, name in ((in_host, si, "in"), (ker_host, sk, "ker"), (out_host, so, "out")):
            if t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != s or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 host tensor of shape {s}")
        if device_buffer.numel() * device_buffer.element_size() < self.host_run_bytes:
            raise ValueError("device_buffer too small")
        _check(self._lib.conv_run_host(self._h, in_host.data_ptr(), ker_host.data_ptr(),
                                       out_host.data_ptr(), device_buffer.data_ptr(),
                                       _stream_handle(stream)))


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _f32():
    import torch
    return torch.float32


_plan_cache = {}


def conv2d(inp, ker, path: str = "auto", out=None, stream=None):
    """Eq. 1 on CUDA tensors (In NCHW [N,C,H+R-1,W+S-1], Ker KCRS) with a
    cached plan per (shape, path, device)."""
    N, C, Hin, Win = inp.shape
    K, C2, R, S = ker.shape
    if C2 != C:
        raise ValueError("channel mismatch between In and Ker")
    key = (N, K, C, Hin - R + 1, Win - S + 1, R, S, path, inp.device.index)
    plan = _plan_cache.get(key)
    if plan is None:
        import torch
        with torch.cuda.device(inp.device):          # the plan binds the current device
            plan = ConvPlan(*key[:7], path=path)
        _plan_cache[key] = plan
    return plan.run(inp, ker, out=out, stream=stream)


# -- the selector's data-movement model (host only; no device needed) ---------
ITER = {"n": 0, "k": 1, "c": 2, "r": 3, "s": 4, "h": 5, "w": 6}


def model_dv(perm: Sequence[str], Nx: dict, T: dict):
    """Sec. 3.2 data volume for tile-loop order ``perm``
    (outermost first, iterator names n,k,c,r,s,h,w).  Returns (In, Ker, Out)."""
    lib = load_library()
    p = (ctypes.c_int * 7)(*[ITER[x] for x in perm])
    order = ["n", "k", "c", "r", "s", "h", "w"]
    n = (ctypes.c_double * 7)(*[float(Nx[x]) for x in order])
    t = (ctypes.c_double * 7)(*[float(T[x]) for x in order])
    dv = (ctypes.c_double * 3)()
    tot = lib.conv_model_dv(p, n, t, dv)
    if tot < 0:
        raise ValueError("invalid model arguments")
    return dv[0], dv[1], dv[2]


def model_dv_matmul(perm: Sequence[str], Nx: dict, T: dict) -> float:
    """Sec. 2.2 matmul model (Eq. 3); iterators i, j, k."""
    lib = load_library()
    ids = {"i": 0, "j": 1, "k": 2}
    p = (ctypes.c_int * 3)(*[ids[x] for x in perm])
    n = (ctypes.c_double * 3)(*[float(Nx[x]) for x in "ijk"])
    t = (ctypes.c_double * 3)(*[float(T[x]) for x in "ijk"])
    tot = lib.conv_model_dv_matmul(p, n, t)
    if tot < 0:
        raise ValueError("invalid model arguments")
    return tot


def model_footprint(T: dict) -> float:
    """Eq. 4 left-hand side."""
    lib = load_library()
    t = (ctypes.c_double * 7)(*[float(T[x]) for x in ["n", "k", "c", "r", "s", "h", "w"]])
    return lib.conv_model_footprint(t)


# B200 as the selector sees it (for offline plans in CPU tests / studies).
B200 = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
