"""Python binding of the B200-native Domain Transform Solver (include/dts.h).

Argument marshalling only: every step of the path runs in the sm_100a kernels of
``libdts_b200.so`` (built in-tree by ``_build.build()`` / ``__graft_entry__.build()``).
There is no CPU fallback: if the library is missing, or there is no sm_100 GPU,
calls raise ``DTSError``.  PyTorch supplies device memory and streams only.

Names follow the C ABI: ``dts_create``, ``dts_solve``, ``dts_solve_ex``,
``dts_destroy`` (+ the test/bench extensions).  Arrays may be torch tensors
(CUDA or CPU) or numpy arrays; they must be float32 and C-contiguous.  Host
arrays are staged by the library itself (include/dts.h).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["DTSError", "dts_create", "dts_create_batch", "dts_solve", "dts_solve_ex", "dts_confidence", "dts_solve_stereo",
           "dts_sr_prepare", "dts_create_ex", "dts_debug_read_windows", "DTS_FILTER_RF", "DTS_FILTER_BOX",
           "dts_destroy",
           "dts_status_string",
           "dts_comm_unique_id", "dts_comm_init", "dts_comm_init_loopback", "dts_comm_destroy",
           "dts_create_band", "band_rows", "band_guide_rows",
           "dts_debug_read", "dts_set_option", "dts_get_option", "options", "dts_profile_enable", "dts_profile_read", "dts_launch_count", "dts_version",
           "Solver", "lib_path", "load_library", "DTS_BUF_DX", "DTS_BUF_DY", "DTS_BUF_SUPPORT",
           "ABI_FUNCTIONS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdts_b200.so")
_lib = None

DTS_BUF_DX, DTS_BUF_DY, DTS_BUF_SUPPORT = 0, 1, 2
DTS_FILTER_RF, DTS_FILTER_BOX = 0, 1

# every symbol declared in include/dts.h
ABI_FUNCTIONS = ["dts_create", "dts_solve", "dts_destroy", "dts_status_string", "dts_last_error_string",
                 "dts_solve_ex", "dts_debug_read", "dts_profile_enable", "dts_profile_read",
                 "dts_launch_count", "dts_comm_unique_id", "dts_comm_init", "dts_comm_init_loopback",
                 "dts_comm_destroy", "dts_create_band", "dts_version", "dts_confidence", "dts_solve_stereo",
                 "dts_sr_prepare", "dts_create_ex", "dts_debug_read_windows", "dts_set_option", "dts_get_option",
                 "dts_create_batch"]


class DTSError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        msg = f"{where}: {dts_status_string(status)}"
        if detail:
            msg += f" ({detail})"
        super().__init__(msg)


class CreateOpts(ctypes.Structure):
    """dts_create_opts (include/dts.h)."""
    _fields_ = [("filter", ctypes.c_int32), ("radius_scale", ctypes.c_float)]


class SolveOpts(ctypes.Structure):
    """dts_solve_opts (include/dts.h)."""
    _fields_ = [("step", ctypes.c_float), ("support_mode", ctypes.c_int32), ("check_inputs", ctypes.c_int32),
                ("resid_inf_out", ctypes.c_void_p)]


class KernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double),
                ("bytes_per_launch", ctypes.c_double)]


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libdts_b200.so (raises DTSError-like RuntimeError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                           f"g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    lib.dts_create.argtypes = [vp, i64, i64, i32, f32, f32, i32, vp, ctypes.POINTER(vp)]
    lib.dts_create_batch.argtypes = [vp, i64, i64, i64, i32, f32, f32, i32, vp, ctypes.POINTER(vp)]
    lib.dts_create_batch.restype = ctypes.c_int
    lib.dts_create.restype = ctypes.c_int
    lib.dts_create_ex.argtypes = [vp, i64, i64, i32, f32, f32, i32, ctypes.POINTER(CreateOpts), vp,
                                  ctypes.POINTER(vp)]
    lib.dts_create_ex.restype = ctypes.c_int
    lib.dts_debug_read_windows.argtypes = [vp, i32, i32, vp]
    lib.dts_debug_read_windows.restype = ctypes.c_int
    lib.dts_solve.argtypes = [vp, vp, i32, vp, f32, i32, vp, vp]
    lib.dts_solve.restype = ctypes.c_int
    lib.dts_solve_ex.argtypes = [vp, vp, i32, vp, f32, i32, vp, vp, ctypes.POINTER(SolveOpts)]
    lib.dts_solve_ex.restype = ctypes.c_int
    lib.dts_confidence.argtypes = [vp, vp, f32, vp, vp, vp]
    lib.dts_confidence.restype = ctypes.c_int
    lib.dts_solve_stereo.argtypes = [vp, vp, vp, f32, i32, vp, vp, vp, f32, f32, vp]
    lib.dts_solve_stereo.restype = ctypes.c_int
    lib.dts_sr_prepare.argtypes = [vp, i64, i64, i32, vp, vp, vp]
    lib.dts_sr_prepare.restype = ctypes.c_int
    lib.dts_set_option.argtypes = [ctypes.c_char_p, i32]
    lib.dts_set_option.restype = ctypes.c_int
    lib.dts_get_option.argtypes = [ctypes.c_char_p]
    lib.dts_get_option.restype = ctypes.c_int32
    lib.dts_destroy.argtypes = [vp]
    lib.dts_destroy.restype = None
    lib.dts_status_string.argtypes = [ctypes.c_int]
    lib.dts_status_string.restype = ctypes.c_char_p
    lib.dts_last_error_string.argtypes = []
    lib.dts_last_error_string.restype = ctypes.c_char_p
    lib.dts_debug_read.argtypes = [vp, ctypes.c_int, vp]
    lib.dts_debug_read.restype = ctypes.c_int
    lib.dts_profile_enable.argtypes = [vp, i32]
    lib.dts_profile_enable.restype = ctypes.c_int
    lib.dts_profile_read.argtypes = [vp, ctypes.POINTER(KernelStat), i32, ctypes.POINTER(i32)]
    lib.dts_profile_read.restype = ctypes.c_int
    lib.dts_launch_count.argtypes = [vp]
    lib.dts_launch_count.restype = i64
    lib.dts_version.argtypes = []
    lib.dts_version.restype = ctypes.c_char_p
    lib.dts_comm_unique_id.argtypes = [vp]
    lib.dts_comm_unique_id.restype = ctypes.c_int
    lib.dts_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    lib.dts_comm_init.restype = ctypes.c_int
    lib.dts_comm_init_loopback.argtypes = [i32, ctypes.POINTER(vp)]
    lib.dts_comm_init_loopback.restype = ctypes.c_int
    lib.dts_comm_destroy.argtypes = [vp]
    lib.dts_comm_destroy.restype = None
    lib.dts_create_band.argtypes = [vp, i64, i64, i64, i64, i32, f32, f32, i32, vp, vp, ctypes.POINTER(vp)]
    lib.dts_create_band.restype = ctypes.c_int
    _lib = lib
    return lib


def dts_status_string(status: int) -> str:
    return load_library().dts_status_string(int(status)).decode()


def dts_version() -> str:
    return load_library().dts_version().decode()


def _check(st: int, where: str):
    if st != 0:
        raise DTSError(st, where, load_library().dts_last_error_string().decode())


def _ptr(a, name: str):
    """Device or host address of a float32 C-contiguous torch tensor / numpy array."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
            raise TypeError(f"{name} must be a C-contiguous float32 array")
        return a.ctypes.data
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.dtype != torch.float32 or not a.is_contiguous():
            raise TypeError(f"{name} must be a contiguous float32 tensor")
        return a.data_ptr()
    raise TypeError(f"{name}: unsupported array type {type(a)}")


def _stream(stream, *arrays):
    if stream is not None:
        return int(stream) if not hasattr(stream, "cuda_stream") else int(stream.cuda_stream)
    try:
        import torch
        if torch.cuda.is_available() and any(getattr(a, "is_cuda", False) for a in arrays):
            return int(torch.cuda.current_stream().cuda_stream)
    except ImportError:  # pragma: no cover
        pass
    return 0


def dts_create(guide, sigma_s: float, sigma_r: float, filter_passes: int = 3, stream=None) -> int:
    """guide: H x W x C float32 (HWC).  Returns an opaque context handle (int)."""
    if len(guide.shape) == 2:
        H, W = guide.shape
        C = 1
    else:
        H, W, C = guide.shape
    ctx = ctypes.c_void_p()
    st = load_library().dts_create(_ptr(guide, "guide"), H, W, C, sigma_s, sigma_r, filter_passes,
                                   _stream(stream, guide), ctypes.byref(ctx))
    _check(st, "dts_create")
    return ctx.value


def dts_create_batch(guides, sigma_s: float, sigma_r: float, filter_passes: int = 3, stream=None) -> int:
    """guides: B x H x W x C (or B x H x W) float32, the images back to back.  One context for
    the B images; solve targets / confidences are B x H x W [x C_t] (include/dts.h)."""
    if len(guides.shape) == 3:
        B, H, W = guides.shape
        C = 1
    else:
        B, H, W, C = guides.shape
    ctx = ctypes.c_void_p()
    st = load_library().dts_create_batch(_ptr(guides, "guides"), B, H, W, C, sigma_s, sigma_r, filter_passes,
                                         _stream(stream, guides), ctypes.byref(ctx))
    _check(st, "dts_create_batch")
    return ctx.value


def dts_create_ex(guide, sigma_s: float, sigma_r: float, filter_passes: int = 3, filter: int = DTS_FILTER_RF,
                  radius_scale: float = 0.0, stream=None) -> int:
    """dts_create with options: filter = DTS_FILTER_BOX builds the box-variant context (reading
    R25); radius_scale 0 selects sqrt(3)."""
    if len(guide.shape) == 2:
        H, W = guide.shape
        C = 1
    else:
        H, W, C = guide.shape
    opts = CreateOpts(int(filter), float(radius_scale))
    ctx = ctypes.c_void_p()
    st = load_library().dts_create_ex(_ptr(guide, "guide"), H, W, C, sigma_s, sigma_r, filter_passes,
                                      ctypes.byref(opts), _stream(stream, guide), ctypes.byref(ctx))
    _check(st, "dts_create_ex")
    return ctx.value


def dts_debug_read_windows(ctx: int, pass_index: int, axis: int, H: int, W: int) -> np.ndarray:
    """Box context: packed windows (lo | hi << 16) of one pass along rows (axis 0) / columns (1)."""
    out = np.empty((H, W), np.uint32)
    _check(load_library().dts_debug_read_windows(ctx, pass_index, axis, out.ctypes.data), "dts_debug_read_windows")
    return out


def dts_solve_ex(ctx: int, target, confidence, lam: float, iterations: int, out, stream=None,
                 step: float = 0.0, support_mode: int = 0, check_inputs: bool = False, resid_inf_out=None):
    """dts_solve with options; resid_inf_out: None or `iterations` float32 (device tensor or host
    array) that receives ||g_k||_inf per iteration (K8)."""
    Ct = _target_channels(target, confidence)
    opts = SolveOpts(step, support_mode, 1 if check_inputs else 0,
                     _ptr(resid_inf_out, "resid_inf_out") if resid_inf_out is not None else None)
    st = load_library().dts_solve_ex(ctx, _ptr(target, "target"), Ct, _ptr(confidence, "confidence"), lam,
                                     iterations, _ptr(out, "out"), _stream(stream, target, confidence, out),
                                     ctypes.byref(opts))
    _check(st, "dts_solve_ex")
    return out


def debug_col_plan(ctx: int, Ct: int) -> dict:
    """FILTER column plan dts_solve uses for C_t on this context (tests / probes)."""
    f = load_library().dts_debug_col_plan
    f.restype = ctypes.c_int32
    f.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    v = (ctypes.c_int32 * 7)()
    if f(ctx, Ct, v) != 0:
        raise DTSError(2, "dts_debug_col_plan")
    return dict(zip(("kind", "CB", "grid", "threads", "HS", "ntiles", "Ls"), list(v)))


def debug_strips(ctx: int) -> dict:
    """Row-strip plan of a context (tests / probes; not part of include/dts.h)."""
    lib = load_library()
    f = lib.dts_debug_strips
    f.restype = ctypes.c_int32
    f.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int32)] * 4
    hs, cb, gr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    L3 = (ctypes.c_int32 * 3)()
    n = f(ctx, ctypes.byref(hs), L3, ctypes.byref(cb), ctypes.byref(gr))
    return {"strips": n, "HS": hs.value, "L": list(L3), "CB": cb.value, "grid": gr.value}


def dts_set_option(name: str, value: int) -> None:
    """Process-wide test / experiment option (include/dts.h); the defaults are the product path."""
    _check(load_library().dts_set_option(name.encode(), int(value)), f"dts_set_option({name}={value})")


def dts_get_option(name: str) -> int:
    return int(load_library().dts_get_option(name.encode()))


class options:
    """``with options(persistent=0): ...`` sets library options and restores them on exit."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = dts_get_option(k)
            dts_set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            dts_set_option(k, v)


def _target_channels(target, confidence) -> int:
    """C_t: the trailing target axis beyond the confidence's shape (H x W, or B x H x W for
    batched contexts); a target shaped like the confidence has one channel."""
    if len(target.shape) == len(confidence.shape):
        return 1
    if len(target.shape) != len(confidence.shape) + 1:
        raise ValueError(f"target shape {tuple(target.shape)} does not extend confidence {tuple(confidence.shape)}")
    return int(target.shape[-1])


def dts_solve(ctx: int, target, confidence, lam: float, iterations: int, out, stream=None):
    """target: H x W (x Ct) float32 HWC; confidence: H x W; out like target (written).  Batched
    contexts (dts_create_batch): B x H x W (x Ct) and B x H x W."""
    Ct = _target_channels(target, confidence)
    st = load_library().dts_solve(ctx, _ptr(target, "target"), Ct, _ptr(confidence, "confidence"), lam,
                                  iterations, _ptr(out, "out"), _stream(stream, target, confidence, out))
    _check(st, "dts_solve")
    return out


def dts_confidence(ctx: int, target, sigma_c: float, conf_out, var_out=None, stream=None):
    """Eq. (7): conf_out = exp(-V / (2 sigma_c^2)), V = DT(t^2) - DT(t)^2 (>= 0) -> var_out.
    target, conf_out, var_out: H x W float32 (device tensors or host arrays)."""
    st = load_library().dts_confidence(ctx, _ptr(target, "target"), sigma_c, _ptr(conf_out, "conf_out"),
                                       _ptr(var_out, "var_out") if var_out is not None else None,
                                       _stream(stream, target, conf_out))
    _check(st, "dts_confidence")
    return conf_out


def dts_solve_stereo(ctx: int, target, confidence, lam: float, iterations: int, out, left, right,
                     gamma: float = 0.001, eps: float = 0.001, stream=None):
    """Eq. (10): stereo refinement of a disparity target with the Charbonnier target term and the
    photometric term gamma (I_L(x) - I_R(x - z))^2; left = the context's guide image, right its
    partner (H x W x C float32 HWC); target, confidence, out: H x W float32."""
    st = load_library().dts_solve_stereo(ctx, _ptr(target, "target"), _ptr(confidence, "confidence"), lam,
                                         iterations, _ptr(out, "out"), _ptr(left, "left"), _ptr(right, "right"),
                                         gamma, eps, _stream(stream, target, confidence, out, left, right))
    _check(st, "dts_solve_stereo")
    return out


def dts_sr_prepare(low, factor: int, target_out=None, conf_out=None, stream=None):
    """Depth-SR front end: bicubic x factor target and Gaussian-bump confidence from an
    h x w low-res depth map.  Returns (target, conf), (h f) x (w f) float32 (numpy for numpy input,
    torch on the input's device otherwise)."""
    h, w = int(low.shape[0]), int(low.shape[1])
    shape = (h * factor, w * factor)
    if target_out is None or conf_out is None:
        if isinstance(low, np.ndarray):
            target_out = np.empty(shape, np.float32) if target_out is None else target_out
            conf_out = np.empty(shape, np.float32) if conf_out is None else conf_out
        else:
            import torch
            target_out = torch.empty(shape, dtype=torch.float32, device=low.device) if target_out is None else target_out
            conf_out = torch.empty(shape, dtype=torch.float32, device=low.device) if conf_out is None else conf_out
    st = load_library().dts_sr_prepare(_ptr(low, "low"), h, w, int(factor), _ptr(target_out, "target_out"),
                                       _ptr(conf_out, "conf_out"), _stream(stream, low, target_out, conf_out))
    _check(st, "dts_sr_prepare")
    return target_out, conf_out


def dts_destroy(ctx: int) -> None:
    if ctx:
        load_library().dts_destroy(ctx)


def dts_debug_read(ctx: int, which: int, H: int, W: int) -> np.ndarray:
    out = np.empty((H, W), np.float32)
    _check(load_library().dts_debug_read(ctx, which, out.ctypes.data), "dts_debug_read")
    return out


def dts_profile_enable(ctx: int, on: bool = True) -> None:
    _check(load_library().dts_profile_enable(ctx, 1 if on else 0), "dts_profile_enable")


def dts_profile_read(ctx: int):
    """{family: {"launches", "total_ms", "bytes_per_launch", "avg_ms"}}"""
    arr = (KernelStat * 32)()
    n = ctypes.c_int32(0)
    _check(load_library().dts_profile_read(ctx, arr, 32, ctypes.byref(n)), "dts_profile_read")
    res = {}
    for i in range(min(n.value, 32)):
        k = arr[i]
        res[k.name.decode()] = {"launches": int(k.launches), "total_ms": float(k.total_ms),
                                "bytes_per_launch": float(k.bytes_per_launch),
                                "avg_ms": float(k.total_ms) / k.launches if k.launches else 0.0}
    return res


def dts_launch_count(ctx: int) -> int:
    return int(load_library().dts_launch_count(ctx))


# ---- row-band mode (multi-GPU) -------------------------------------------------

def band_rows(H: int, nranks: int, rank: int):
    """Rows [row0, row1) owned by `rank` when H rows are split over `nranks` ranks:
    row0 = floor(rank H / nranks)."""
    if not (0 <= rank < nranks):
        raise ValueError("rank out of range")
    return (rank * H) // nranks, ((rank + 1) * H) // nranks


def band_guide_rows(H: int, row0: int, row1: int):
    """Guide rows a band context needs: its rows plus one halo row above / below where
    a neighbouring band exists (include/dts.h dts_create_band)."""
    return max(row0 - 1, 0), min(row1 + 1, H)


def dts_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().dts_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "dts_comm_unique_id")
    return buf.raw


def dts_comm_init(uid: bytes, rank: int, nranks: int) -> int:
    if len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    comm = ctypes.c_void_p()
    _check(load_library().dts_comm_init(ctypes.cast(buf, ctypes.c_void_p), rank, nranks, ctypes.byref(comm)),
           "dts_comm_init")
    return comm.value


def dts_comm_init_loopback(nranks: int):
    arr = (ctypes.c_void_p * nranks)()
    _check(load_library().dts_comm_init_loopback(nranks, arr), "dts_comm_init_loopback")
    return [arr[i] for i in range(nranks)]


def dts_comm_destroy(comm: int) -> None:
    if comm:
        load_library().dts_comm_destroy(comm)


def dts_create_band(guide_with_halo, H_total: int, row0: int, rows: int, sigma_s: float, sigma_r: float,
                    filter_passes: int = 3, comm=None, stream=None) -> int:
    """guide_with_halo: the band's guide rows plus halo rows (see band_guide_rows)."""
    if len(guide_with_halo.shape) == 2:
        W, C = guide_with_halo.shape[1], 1
    else:
        W, C = guide_with_halo.shape[1], guide_with_halo.shape[2]
    ctx = ctypes.c_void_p()
    st = load_library().dts_create_band(_ptr(guide_with_halo, "guide"), H_total, row0, rows, W, C, sigma_s,
                                        sigma_r, filter_passes, comm, _stream(stream, guide_with_halo),
                                        ctypes.byref(ctx))
    _check(st, "dts_create_band")
    return ctx.value


class Solver:
    """Thin RAII wrapper: ``Solver(guide, sigma_s, sigma_r, N).solve(t, c, lam, iters)``."""

    def __init__(self, guide, sigma_s: float, sigma_r: float, filter_passes: int = 3, stream=None,
                 filter: int = DTS_FILTER_RF, radius_scale: float = 0.0, batched: bool = False):
        """batched: guide is B x H x W [x C], one context for the B images (dts_create_batch)."""
        self.filter = filter
        if batched:
            if filter != DTS_FILTER_RF:
                raise ValueError("batched contexts use the recursive filter")
            # the stacked image (debug reads return B*H x W)
            self.H, self.W = int(guide.shape[0]) * int(guide.shape[1]), int(guide.shape[2])
            self.ctx = dts_create_batch(guide, sigma_s, sigma_r, filter_passes, stream)
            return
        self.H, self.W = int(guide.shape[0]), int(guide.shape[1])
        if filter == DTS_FILTER_RF:
            self.ctx = dts_create(guide, sigma_s, sigma_r, filter_passes, stream)
        else:
            self.ctx = dts_create_ex(guide, sigma_s, sigma_r, filter_passes, filter, radius_scale, stream)

    def solve(self, target, confidence, lam: float, iterations: int, out=None, stream=None, **opts):
        if out is None:
            if isinstance(target, np.ndarray):
                out = np.empty_like(target)
            else:
                import torch
                out = torch.empty_like(target)
        if opts:
            return dts_solve_ex(self.ctx, target, confidence, lam, iterations, out, stream, **opts)
        return dts_solve(self.ctx, target, confidence, lam, iterations, out, stream)

    def solve_stereo(self, target, confidence, lam: float, iterations: int, left, right, gamma: float = 0.001,
                     eps: float = 0.001, out=None, stream=None):
        if out is None:
            if isinstance(target, np.ndarray):
                out = np.empty_like(target)
            else:
                import torch
                out = torch.empty_like(target)
        return dts_solve_stereo(self.ctx, target, confidence, lam, iterations, out, left, right, gamma, eps, stream)

    def confidence(self, target, sigma_c: float, out=None, var_out=None, stream=None):
        if out is None:
            if isinstance(target, np.ndarray):
                out = np.empty_like(target)
            else:
                import torch
                out = torch.empty_like(target)
        return dts_confidence(self.ctx, target, sigma_c, out, var_out, stream)

    def read(self, which: int) -> np.ndarray:
        return dts_debug_read(self.ctx, which, self.H, self.W)

    def windows(self, pass_index: int, axis: int) -> np.ndarray:
        return dts_debug_read_windows(self.ctx, pass_index, axis, self.H, self.W)

    def close(self):
        if self.ctx:
            dts_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
