"""fp64 CPU oracle for the Domain Transform Solver (arXiv 1805.04590).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1805_04590_b200`` never imports it, and
it shares no code with the CUDA path: the arithmetic lives in ``dts_oracle.c``
(plain loops, double precision); this module only marshals numpy arrays.

Functions (each cites the passage its C routine follows; see dts_oracle.c):
  distances(guide, sigma_s, sigma_r)            O1  P:231-240 (Eqs. 8-9)
  sigmas(sigma_s, N)                            O2  pass schedule (reading R5)
  rf1d(x, A)                                    O3  recursive filter, causal + anticausal (R4)
  dtf(X, dx, dy, sigma_s, N)                    O4  X then Y passes
  support(dx, dy, sigma_s, mode)                O5  S = sum_j W_ij
  solve(guide, target, conf, ...)               O6  Eq. (3) gradient descent
  confidence(guide, target, ..., sigma_c)       O7  Eq. (7) edge-aware variance confidence
  solve_stereo(left, right, target, conf, ...)  O8  Eq. (10) stereo refinement, Charbonnier target
  sr_prepare(low, factor)                       O9  depth-SR front end: bicubic target, bump confidence
  box_increments(guide, sigma_s, sigma_r)       O10a fixed-point DT increments (reading R25)
  box_radius(radius_scale, sigma)               O10  R = floor(r * 2^16)
  box_tables(guide, ..., N, radius_scale)       O10b box windows of every pass + support
  box_dtf(X, guide, ..., N, radius_scale)       O10d 2-D box mean, X then Y per pass
  solve_box(guide, target, conf, ...)           O10e Eq. (3) iteration with the box mean

Parity status: O1, O3, O4, O5, O6, O7, O8, O9 and O10 are pinned by tests/test_oracle_pins.py
(worked examples, dense triangular matrices, closed forms, brute force,
reductions); the whole solve is NOT pinned against the paper's own outputs,
which it never prints ("parity unpinned vs the paper").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dts_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libdts_oracle.so")
_lib = None

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_float_p = ctypes.POINTER(ctypes.c_float)


def build(force: bool = False) -> str:
    """Compile dts_oracle.c into oracle/libdts_oracle.so (gcc, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
               "-shared", "-fPIC", "-o", _LIB_PATH, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB_PATH)
    i64, i32, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    lib.dts_oracle_distances.argtypes = [_c_float_p, i64, i64, i32, dbl, dbl, _c_double_p, _c_double_p]
    lib.dts_oracle_distances.restype = ctypes.c_int
    lib.dts_oracle_sigmas.argtypes = [dbl, i32, _c_double_p]
    lib.dts_oracle_sigmas.restype = None
    lib.dts_oracle_rf1d.argtypes = [_c_double_p, _c_double_p, i64, i64]
    lib.dts_oracle_rf1d.restype = None
    lib.dts_oracle_dtf.argtypes = [_c_double_p, i64, i64, i32, _c_double_p, _c_double_p, dbl, i32]
    lib.dts_oracle_dtf.restype = ctypes.c_int
    lib.dts_oracle_support.argtypes = [_c_double_p, _c_double_p, i64, i64, dbl, i32, _c_double_p]
    lib.dts_oracle_support.restype = ctypes.c_int
    lib.dts_oracle_solve.argtypes = [_c_float_p, i64, i64, i32, dbl, dbl, i32,
                                     _c_float_p, i32, _c_float_p, dbl, dbl, i32, i32,
                                     _c_double_p, _c_double_p]
    lib.dts_oracle_solve.restype = ctypes.c_int
    lib.dts_oracle_confidence.argtypes = [_c_float_p, i64, i64, i32, dbl, dbl, i32, _c_float_p, dbl,
                                          _c_double_p, _c_double_p]
    lib.dts_oracle_confidence.restype = ctypes.c_int
    lib.dts_oracle_solve_stereo.argtypes = [_c_float_p, _c_float_p, i64, i64, i32, dbl, dbl, i32, _c_float_p,
                                            _c_float_p, dbl, dbl, i32, dbl, dbl, i32, _c_double_p]
    lib.dts_oracle_solve_stereo.restype = ctypes.c_int
    lib.dts_oracle_sr_prepare.argtypes = [_c_float_p, i64, i64, i32, _c_double_p, _c_double_p]
    lib.dts_oracle_sr_prepare.restype = ctypes.c_int
    c_i64_p = ctypes.POINTER(ctypes.c_int64)
    c_i32_p = ctypes.POINTER(ctypes.c_int32)
    flt = ctypes.c_float
    lib.dts_oracle_box_increments.argtypes = [_c_float_p, i64, i64, i32, flt, flt, c_i64_p, c_i64_p]
    lib.dts_oracle_box_increments.restype = ctypes.c_int
    lib.dts_oracle_box_radius.argtypes = [dbl, dbl]
    lib.dts_oracle_box_radius.restype = i64
    lib.dts_oracle_box_tables.argtypes = [_c_float_p, i64, i64, i32, flt, flt, i32, dbl,
                                          c_i32_p, c_i32_p, c_i32_p, c_i32_p, _c_double_p]
    lib.dts_oracle_box_tables.restype = ctypes.c_int
    lib.dts_oracle_box_dtf.argtypes = [_c_double_p, i64, i64, i32, _c_float_p, i32, flt, flt, i32, dbl]
    lib.dts_oracle_box_dtf.restype = ctypes.c_int
    lib.dts_oracle_solve_box.argtypes = [_c_float_p, i64, i64, i32, flt, flt, i32, dbl, _c_float_p, i32,
                                         _c_float_p, dbl, dbl, i32, i32, _c_double_p]
    lib.dts_oracle_solve_box.restype = ctypes.c_int
    lib.dts_oracle_num_threads.argtypes = []
    lib.dts_oracle_num_threads.restype = ctypes.c_int
    lib.dts_oracle_set_threads.argtypes = [ctypes.c_int]
    lib.dts_oracle_set_threads.restype = None
    _lib = lib
    return lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(t)


def num_threads() -> int:
    return _load().dts_oracle_num_threads()


def set_threads(n: int) -> None:
    _load().dts_oracle_set_threads(int(n))


def distances(guide, sigma_s: float, sigma_r: float):
    """O1: (d_x, d_y), each H x W float64; +inf on the first column / row."""
    g = _f32(guide)
    if g.ndim == 2:
        g = g[:, :, None]
    H, W, C = g.shape
    dx = np.empty((H, W), np.float64)
    dy = np.empty((H, W), np.float64)
    st = _load().dts_oracle_distances(_p(g, _c_float_p), H, W, C, sigma_s, sigma_r,
                                      _p(dx, _c_double_p), _p(dy, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_distances failed ({st})")
    return dx, dy


def sigmas(sigma_s: float, N: int):
    """O2: per-pass sigma_i, i = 1..N."""
    out = np.empty(N, np.float64)
    _load().dts_oracle_sigmas(sigma_s, N, _p(out, _c_double_p))
    return out


def rf1d(x, A):
    """O3: one causal + anticausal recursive-filter pass of a 1-D signal."""
    z = _f64(x).copy()
    a = _f64(A)
    assert a.shape == z.shape and z.ndim == 1
    _load().dts_oracle_rf1d(_p(z, _c_double_p), _p(a, _c_double_p), z.shape[0], 1)
    return z


def dtf(X, dx, dy, sigma_s: float, N: int):
    """O4: DTF of an H x W (or Ct x H x W planar) array; returns a new array."""
    Z = _f64(X).copy()
    squeeze = Z.ndim == 2
    if squeeze:
        Z = Z[None]
    Ct, H, W = Z.shape
    dxa, dya = _f64(dx), _f64(dy)
    st = _load().dts_oracle_dtf(_p(Z, _c_double_p), H, W, Ct, _p(dxa, _c_double_p),
                                _p(dya, _c_double_p), sigma_s, N)
    if st:
        raise ValueError(f"dts_oracle_dtf failed ({st})")
    return Z[0] if squeeze else Z


def support(dx, dy, sigma_s: float, mode: int = 0):
    """O5: S = s_x * s_y (mode 0) or S = 1 (mode 1)."""
    dxa, dya = _f64(dx), _f64(dy)
    H, W = dxa.shape
    S = np.empty((H, W), np.float64)
    st = _load().dts_oracle_support(_p(dxa, _c_double_p), _p(dya, _c_double_p), H, W,
                                    sigma_s, mode, _p(S, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_support failed ({st})")
    return S


def solve(guide, target, confidence, sigma_s: float, sigma_r: float, N: int,
          lam: float, iters: int, step: float = 0.99, support_mode: int = 0,
          diagnostics: bool = False):
    """O6: the DTS gradient-descent solve.  Returns out (H x W x Ct float64; H x W if the
    target was 2-D) and, if diagnostics, an iters x 4 array [|g|_inf, |g|_2, Fhat, Eq]."""
    g = _f32(guide)
    if g.ndim == 2:
        g = g[:, :, None]
    t = _f32(target)
    squeeze = t.ndim == 2
    if squeeze:
        t = t[:, :, None]
    c = _f32(confidence)
    H, W, Cg = g.shape
    assert t.shape[:2] == (H, W) and c.shape == (H, W)
    Ct = t.shape[2]
    out = np.empty((H, W, Ct), np.float64)
    diag = np.zeros((max(iters, 1), 4), np.float64)
    st = _load().dts_oracle_solve(_p(g, _c_float_p), H, W, Cg, sigma_s, sigma_r, N,
                                  _p(t, _c_float_p), Ct, _p(c, _c_float_p), lam, step,
                                  iters, support_mode, _p(out, _c_double_p),
                                  _p(diag, _c_double_p) if diagnostics else None)
    if st:
        raise ValueError(f"dts_oracle_solve failed ({st})")
    res = out[:, :, 0] if squeeze else out
    if diagnostics:
        return res, diag[:iters]
    return res


def confidence(guide, target, sigma_s: float, sigma_r: float, N: int, sigma_c: float):
    """O7: Eq. (7) confidence c = exp(-V / (2 sigma_c^2)), V = DTF(t^2) - DTF(t)^2 clamped at 0.
    Returns (c, V), each H x W float64."""
    g = _f32(guide)
    if g.ndim == 2:
        g = g[:, :, None]
    t = _f32(target)
    H, W, Cg = g.shape
    assert t.shape == (H, W)
    c = np.empty((H, W), np.float64)
    v = np.empty((H, W), np.float64)
    st = _load().dts_oracle_confidence(_p(g, _c_float_p), H, W, Cg, sigma_s, sigma_r, N,
                                       _p(t, _c_float_p), sigma_c, _p(c, _c_double_p), _p(v, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_confidence failed ({st})")
    return c, v


def solve_stereo(left, right, target, confidence, sigma_s: float, sigma_r: float, N: int, lam: float,
                 iters: int, gamma: float, eps: float = 1e-3, step: float = 0.99, support_mode: int = 0):
    """O8: Eq. (10) stereo refinement with the Charbonnier target term.  left (the guide) and
    right: H x W x Cg; target, confidence: H x W.  Returns z (H x W float64)."""
    g = _f32(left)
    if g.ndim == 2:
        g = g[:, :, None]
    rr = _f32(right)
    if rr.ndim == 2:
        rr = rr[:, :, None]
    t = _f32(target)
    c = _f32(confidence)
    H, W, Cg = g.shape
    assert rr.shape == g.shape and t.shape == (H, W) and c.shape == (H, W)
    out = np.empty((H, W), np.float64)
    st = _load().dts_oracle_solve_stereo(_p(g, _c_float_p), _p(rr, _c_float_p), H, W, Cg, sigma_s, sigma_r, N,
                                         _p(t, _c_float_p), _p(c, _c_float_p), lam, step, iters, gamma, eps,
                                         support_mode, _p(out, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_solve_stereo failed ({st})")
    return out


def sr_prepare(low, factor: int):
    """O9: (target, confidence), each (h f) x (w f) float64, from an h x w low-res depth map."""
    lo = _f32(low)
    h, w = lo.shape
    H, W = h * factor, w * factor
    t = np.empty((H, W), np.float64)
    c = np.empty((H, W), np.float64)
    st = _load().dts_oracle_sr_prepare(_p(lo, _c_float_p), h, w, int(factor), _p(t, _c_double_p), _p(c, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_sr_prepare failed ({st})")
    return t, c


SQRT3 = float(np.sqrt(3.0))


def _guide3(guide):
    g = _f32(guide)
    return g[:, :, None] if g.ndim == 2 else g


def box_increments(guide, sigma_s: float, sigma_r: float):
    """O10a: fixed-point DT increments (qx, qy), each H x W int64 (d in fp32, times 2^16,
    rounded half-even, capped at 2^30; qx[:, 0] = qy[0, :] = 0).  Reading R25."""
    g = _guide3(guide)
    H, W, C = g.shape
    qx = np.empty((H, W), np.int64)
    qy = np.empty((H, W), np.int64)
    c_i64_p = ctypes.POINTER(ctypes.c_int64)
    st = _load().dts_oracle_box_increments(_p(g, _c_float_p), H, W, C, float(np.float32(sigma_s)),
                                           float(np.float32(sigma_r)), _p(qx, c_i64_p), _p(qy, c_i64_p))
    if st:
        raise ValueError(f"dts_oracle_box_increments failed ({st})")
    return qx, qy


def box_radius(radius_scale: float, sigma: float) -> int:
    """R = floor(radius_scale * sigma * 2^16) (fixed-point box radius, reading R25)."""
    return int(_load().dts_oracle_box_radius(float(radius_scale), float(sigma)))


def box_tables(guide, sigma_s: float, sigma_r: float, N: int, radius_scale: float = SQRT3):
    """O10b: windows of every pass and the support.  Returns (lox, hix, loy, hiy, S):
    lo/hi offsets N x H x W int32 (window of pixel i along the line = [i - lo, i + hi]),
    S = |N^x| |N^y| at r = radius_scale * sigma_s, H x W float64.  sigma_s and sigma_r
    are taken as float32 (the ABI's type)."""
    g = _guide3(guide)
    H, W, C = g.shape
    lox, hix, loy, hiy = (np.empty((N, H, W), np.int32) for _ in range(4))
    S = np.empty((H, W), np.float64)
    c_i32_p = ctypes.POINTER(ctypes.c_int32)
    st = _load().dts_oracle_box_tables(_p(g, _c_float_p), H, W, C, float(np.float32(sigma_s)),
                                       float(np.float32(sigma_r)), N, float(radius_scale),
                                       _p(lox, c_i32_p), _p(hix, c_i32_p), _p(loy, c_i32_p), _p(hiy, c_i32_p),
                                       _p(S, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_box_tables failed ({st})")
    return lox, hix, loy, hiy, S


def box_dtf(X, guide, sigma_s: float, sigma_r: float, N: int, radius_scale: float = SQRT3):
    """O10d: 2-D box mean of X (H x W, or Ct x H x W planar), float64 result."""
    x = np.array(X, dtype=np.float64, copy=True, order="C")
    planes = x[None] if x.ndim == 2 else x
    g = _guide3(guide)
    H, W, C = g.shape
    assert planes.shape[1:] == (H, W)
    st = _load().dts_oracle_box_dtf(_p(planes, _c_double_p), H, W, planes.shape[0], _p(g, _c_float_p), C,
                                    float(np.float32(sigma_s)), float(np.float32(sigma_r)), N, float(radius_scale))
    if st:
        raise ValueError(f"dts_oracle_box_dtf failed ({st})")
    return planes[0] if x.ndim == 2 else planes


def solve_box(guide, target, confidence, sigma_s: float, sigma_r: float, N: int, lam: float, iters: int,
              step: float = 0.99, support_mode: int = 0, radius_scale: float = SQRT3):
    """O10e: the DTS iteration with the box mean and the box support.  Returns H x W x Ct
    (H x W for a 2-D target) float64."""
    g = _guide3(guide)
    t = _f32(target)
    squeeze = t.ndim == 2
    if squeeze:
        t = t[:, :, None]
    c = _f32(confidence)
    H, W, Cg = g.shape
    assert t.shape[:2] == (H, W) and c.shape == (H, W)
    Ct = t.shape[2]
    out = np.empty((H, W, Ct), np.float64)
    st = _load().dts_oracle_solve_box(_p(g, _c_float_p), H, W, Cg, float(np.float32(sigma_s)),
                                      float(np.float32(sigma_r)), N, float(radius_scale), _p(t, _c_float_p), Ct,
                                      _p(c, _c_float_p), lam, step, iters, support_mode, _p(out, _c_double_p))
    if st:
        raise ValueError(f"dts_oracle_solve_box failed ({st})")
    return out[:, :, 0] if squeeze else out
