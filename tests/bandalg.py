"""Row-band algebra of one column pass in plain fp64 numpy (tests only).

An independent restatement of the exchange the CUDA row-band mode performs
(DESIGN.md "Multi-GPU"): each band of rows [lo, hi) of a column summarises its
causal + anticausal recursive-filter pass (R4) as the 5-tuple
    y[hi-1] = A c + B,            z[lo] = Z0 + S c + Q e
in the unknown carries c = y[lo-1] (from above) and e = z[hi] (from below); the
tuples are gathered in band order, the carries composed
    c_{k+1} = A_k c_k + B_k (c_0 = 0),   e_{k-1} = Z0_k + S_k c_k + Q_k e_k (e_last = 0),
and each band finishes with its exact carries.  Nothing here calls the oracle or
the CUDA library.
"""
import numpy as np


def band_parts(x, A, lo, hi, A_below):
    """Per-band quantities for x[lo:hi] with coefficients A[lo:hi] and the link
    coefficient A_below between row hi-1 and row hi (0 at the image bottom)."""
    n = hi - lo
    y0 = np.zeros(n)
    y1 = np.zeros(n)
    p0, p1 = 0.0, 1.0
    for i in range(n):
        a = A[lo + i]
        p0 = a * p0 + (1 - a) * x[lo + i]
        p1 = a * p1
        y0[i], y1[i] = p0, p1
    z0 = np.zeros(n)
    S = np.zeros(n)
    Q = np.zeros(n)
    q0, qs, qq = 0.0, 0.0, 1.0
    for i in range(n - 1, -1, -1):
        an = A_below if i == n - 1 else A[lo + i + 1]
        q0 = an * q0 + (1 - an) * y0[i]
        qs = an * qs + (1 - an) * y1[i]
        qq = an * qq
        z0[i], S[i], Q[i] = q0, qs, qq
    tup = np.array([y1[-1], y0[-1], z0[0], S[0], Q[0]])  # A, B, Z0, S, Q
    return tup, (y0, y1, z0, S, Q)


def compose(tuples):
    """Carries (c_k, e_k) of every band from the gathered tuples (band order)."""
    P = len(tuples)
    c = np.zeros(P)
    for k in range(P - 1):
        A, B = tuples[k][0], tuples[k][1]
        c[k + 1] = A * c[k] + B
    e = np.zeros(P)
    for k in range(P - 1, 0, -1):
        Z0, S, Q = tuples[k][2], tuples[k][3], tuples[k][4]
        e[k - 1] = Z0 + S * c[k] + Q * e[k]
    return c, e


def finish(parts, c, e):
    y0, y1, z0, S, Q = parts
    return z0 + S * c + Q * e


# ---- edge fix-up scheme ("Edge fix-up scheme") ----------------------
def zero_carry_pass(x, A, lo, hi, A_below):
    """Causal + anticausal pass of rows [lo, hi) with zero carries: y[lo-1] = 0 enters
    through A[lo], z[hi] = 0 enters through A_below.  Returns (y0, z0)."""
    n = hi - lo
    y = np.zeros(n)
    p = 0.0
    for i in range(n):
        a = A[lo + i]
        p = a * p + (1 - a) * x[lo + i]
        y[i] = p
    z = np.zeros(n)
    q = 0.0
    for i in range(n - 1, -1, -1):
        an = A[lo + i + 1] if i + 1 < n else A_below
        q = an * q + (1 - an) * y[i]
        z[i] = q
    return y, z


def edge_profiles(A, lo, hi, A_below, L):
    """Gamma (anticausal response of G_k = prod_{j<=k} A[lo+j]) on the top L rows and
    Theta_k = prod_{j=k+1..hi} a_j (a_hi = A_below) on the bottom L rows."""
    G = np.cumprod(A[lo:lo + L])
    gam = np.zeros(L)
    dz = 0.0
    for k in range(L - 1, -1, -1):
        an = A[lo + k + 1]
        dz = an * (dz - G[k]) + G[k]
        gam[k] = dz
    theta = np.zeros(L)
    th = A_below
    for k in range(hi - 1, hi - L - 1, -1):
        theta[k - (hi - L)] = th
        th *= A[k]
    return G, gam, theta


def edge_scheme(x, A, cuts, L):
    """The banded pass by the edge scheme: zero-carry pass per band, exchange of (y0 at the
    band's last row, z0 at its first row, Gamma_0), corrections on the L edge rows."""
    P = len(cuts) - 1
    H = cuts[-1]
    ys, zs, prof = [], [], []
    for k in range(P):
        lo, hi = cuts[k], cuts[k + 1]
        below = A[hi] if hi < H else 0.0
        y0, z0 = zero_carry_pass(x, A, lo, hi, below)
        ys.append(y0)
        zs.append(z0)
        prof.append(edge_profiles(A, lo, hi, below, L))
    out = []
    for k in range(P):
        z = zs[k].copy()
        c = ys[k - 1][-1] if k > 0 else 0.0
        e = zs[k + 1][0] + ys[k][-1] * prof[k + 1][1][0] if k + 1 < P else 0.0
        _, gam, theta = prof[k]
        z[:L] += c * gam
        z[-L:] += e * theta
        out.append(z)
    return np.concatenate(out)


def edge_scheme_cut(x, A, cuts, L, fix_carry=True):
    """The edge scheme with the link below each band cut (a_hi taken as 0 in the zero-carry
    pass, as the single-context column kernel does at its last row).  The cut pass's output
    at the band's last row is y0 itself and at its first row z0, so the exchanged values are
    read from the output; the bottom carry becomes z_hi - y0(hi - 1) on the same Theta."""
    P = len(cuts) - 1
    H = cuts[-1]
    zs, prof = [], []
    for k in range(P):
        lo, hi = cuts[k], cuts[k + 1]
        below = A[hi] if hi < H else 0.0
        _, z0 = zero_carry_pass(x, A, lo, hi, 0.0)  # cut below
        zs.append(z0)
        prof.append(edge_profiles(A, lo, hi, below, L))
    out = []
    for k in range(P):
        z = zs[k].copy()
        ylast = zs[k][-1]  # = y0 at the last row (the cut makes z = y there)
        c = zs[k - 1][-1] if k > 0 else 0.0
        e = (zs[k + 1][0] + ylast * prof[k + 1][1][0]) - (ylast if fix_carry else 0.0) if k + 1 < P else 0.0
        _, gam, theta = prof[k]
        z[:L] += c * gam
        z[-L:] += e * theta
        out.append(z)
    return np.concatenate(out)
