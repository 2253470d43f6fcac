"""Independent dense-matrix forms used to pin the oracle (tests only).

These are the closed-form products of the recursive filter, NOT the
recurrences: the causal pass is the lower-triangular matrix
    L_kk = 1 - A_k (L_00 = 1),  L_km = (1 - A_m) * prod_{j=m+1..k} A_j   (m < k)
and the anticausal pass the upper-triangular matrix
    U_kk = 1 - A_{k+1} (U_{n-1,n-1} = 1),  U_km = (1 - A_{m+1}) * prod_{j=k+1..m} A_j   (m > k)
(SURVEY.md 8(c) "What pins each part"), so a 1-D pass is U @ L and the 2-D
edge-aware mean of N passes is K = Col_N Row_N ... Col_1 Row_1.
Nothing here calls the oracle.
"""
import numpy as np


def lower(A):
    A = np.asarray(A, np.float64)
    n = len(A)
    L = np.zeros((n, n))
    for k in range(n):
        for m in range(k + 1):
            coef = 1.0 if m == 0 else 1.0 - A[m]
            L[k, m] = coef * np.prod(A[m + 1:k + 1])
    return L


def upper(A):
    A = np.asarray(A, np.float64)
    n = len(A)
    Aext = np.append(A, 0.0)  # A_n = 0: nothing beyond the last sample
    U = np.zeros((n, n))
    for k in range(n):
        for m in range(k, n):
            U[k, m] = (1.0 - Aext[m + 1]) * np.prod(Aext[k + 1:m + 1])
    return U


def pass1d(A):
    return upper(A) @ lower(A)


def row_operator(Ax):
    """Block-diagonal operator filtering every row of an H x W image (row-major vector)."""
    H, W = Ax.shape
    M = np.zeros((H * W, H * W))
    for r in range(H):
        M[r * W:(r + 1) * W, r * W:(r + 1) * W] = pass1d(Ax[r])
    return M


def col_operator(Ay):
    H, W = Ay.shape
    M = np.zeros((H * W, H * W))
    for c in range(W):
        P = pass1d(Ay[:, c])
        idx = np.arange(H) * W + c
        M[np.ix_(idx, idx)] = P
    return M


def dtf_operator(dx, dy, sigmas):
    """K for the N-pass 2-D filter, coefficients a_i^d = exp(-sqrt2 d / sigma_i)."""
    H, W = dx.shape
    K = np.eye(H * W)
    for s in sigmas:
        Ax = np.exp(-np.sqrt(2.0) * dx / s)
        Ay = np.exp(-np.sqrt(2.0) * dy / s)
        K = col_operator(Ay) @ row_operator(Ax) @ K
    return K


def edge_free_kernel(a, half):
    """Interior impulse response of one edge-free pass: (1-a)/(1+a) a^|k|, k = -half..half."""
    k = np.arange(-half, half + 1)
    return (1 - a) / (1 + a) * a ** np.abs(k)
