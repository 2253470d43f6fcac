"""Seeded synthetic DTS workloads C0..C4 (BASELINE.json "configs", 0-based).

Everything here is input synthesis: scene geometry, colours, noise, outliers.
Per-pixel random draws come from independent streams per block of BLOCK rows,
seeded by (seed, stream, block), so any row range of a workload can be produced
on its own (row-band sharding) and the result never depends on thread count.

Stand-ins: C1 for Middlebury stereo refinement, C2 for the
Ferstl 16x depth-SR benchmark, C3 for the multi-channel claim
(P:76), C4 for the 100-MP, 16-band satellite motivation.  None of those
datasets' items is reproduced; the scenes are random shapes.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK = 64  # rows per independent random stream

# stream ids
_S_GUIDE_NOISE = 1
_S_TARGET_NOISE = 2
_S_OUTLIER = 3
_S_CONF = 4


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    W: int
    H: int
    Cg: int
    Ct: int
    sigma_s: float
    sigma_r: float
    N: int
    lam: float
    iters: int
    seed: int
    batch: int = 1
    scene: str = "rects"

    @property
    def pixels(self) -> int:
        return self.W * self.H * self.batch

    @property
    def mpix_iter(self) -> float:
        return self.pixels * self.iters / 1e6


# BASELINE.json configs; lambda for C1-C4 is the paper's 0.99 (reading R10)
CONFIGS = {
    "C0": Config("C0", 64, 48, 3, 1, 8.0, 0.2, 3, 1.0, 20, 0, 1, "rects"),
    "C1": Config("C1", 1400, 1000, 3, 1, 16.0, 0.1, 3, 0.99, 50, 1, 1, "stereo"),
    "C2": Config("C2", 1376, 1024, 3, 1, 32.0, 0.08, 3, 0.99, 100, 2, 1, "sr16"),
    "C3": Config("C3", 3840, 2160, 3, 3, 24.0, 0.15, 3, 0.99, 30, 30, 8, "blur"),
    "C4": Config("C4", 10000, 10000, 16, 1, 64.0, 0.2, 3, 0.99, 20, 4, 1, "satellite"),
}


def _rng(seed: int, stream: int, block: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(stream), int(block)])


def _blocks(r0: int, r1: int):
    """(block index, lo, hi) covering rows [r0, r1), aligned to BLOCK."""
    b = r0 // BLOCK
    while b * BLOCK < r1:
        lo, hi = b * BLOCK, (b + 1) * BLOCK
        yield b, lo, hi
        b += 1


def _per_block(fn, r0, r1, nthreads=None):
    """Run fn(block, lo, hi) for every block overlapping [r0, r1) in parallel."""
    blocks = list(_blocks(r0, r1))
    nthreads = nthreads or min(len(blocks), os.cpu_count() or 1)
    if nthreads <= 1 or len(blocks) <= 1:
        for b in blocks:
            fn(*b)
        return
    with ThreadPoolExecutor(nthreads) as ex:
        list(ex.map(lambda a: fn(*a), blocks))


def _block_noise(seed, stream, b, lo, hi, r0, r1, W, C, scale):
    """Noise rows of block b restricted to [r0, r1); the full block is always drawn."""
    n = _rng(seed, stream, b).standard_normal((hi - lo, W, C), dtype=np.float32)
    n *= np.float32(scale)
    return n[max(r0, lo) - lo: min(r1, hi) - lo]


# ---------------------------------------------------------------------------
# scene geometry: label maps
# ---------------------------------------------------------------------------

def _rects_scene(cfg: Config):
    rng = np.random.default_rng([cfg.seed, 0])
    W, H = cfg.W, cfg.H
    rects = []
    for _ in range(6):
        w = int(rng.integers(4, W // 2 + 1))
        h = int(rng.integers(4, H // 2 + 1))
        x0 = int(rng.integers(0, W - w + 1))
        y0 = int(rng.integers(0, H - h + 1))
        rects.append((x0, y0, w, h))
    colours = rng.uniform(0, 1, (7, cfg.Cg)).astype(np.float32)  # 0 = background
    values = rng.uniform(0, 1, 7).astype(np.float32)
    return rects, colours, values


def _rects_labels(rects, r0, r1, W):
    lab = np.zeros((r1 - r0, W), np.int32)
    for i, (x0, y0, w, h) in enumerate(rects):
        a, b = max(y0, r0), min(y0 + h, r1)
        if a < b:
            lab[a - r0:b - r0, x0:x0 + w] = i + 1
    return lab


def _ellipse_scene(cfg: Config, seed: int, n: int = 40):
    rng = np.random.default_rng([seed, 0])
    W, H = cfg.W, cfg.H
    cx = rng.uniform(0, W, n)
    cy = rng.uniform(0, H, n)
    ax = rng.uniform(W / 50, W / 8, n)
    by = rng.uniform(W / 50, W / 8, n)
    th = rng.uniform(0, np.pi, n)
    # region 0 = background; colour = base + linear gradient (per channel, per pixel)
    base = rng.uniform(0, 1, (n + 1, cfg.Cg))
    grad = rng.uniform(-0.5, 0.5, (n + 1, 2, cfg.Cg)) / (W / 8)
    ctr = np.concatenate([[[W / 2, H / 2]], np.stack([cx, cy], 1)], 0)
    return dict(cx=cx, cy=cy, ax=ax, by=by, th=th, base=base, grad=grad, ctr=ctr, rng=rng)


def _ellipse_labels(sc, r0, r1, W):
    lab = np.zeros((r1 - r0, W), np.int32)
    for i in range(len(sc["cx"])):
        cx, cy, a, b, t = sc["cx"][i], sc["cy"][i], sc["ax"][i], sc["by"][i], sc["th"][i]
        R = max(a, b)
        ya, yb = max(int(np.floor(cy - R)), r0), min(int(np.ceil(cy + R)) + 1, r1)
        xa, xb = max(int(np.floor(cx - R)), 0), min(int(np.ceil(cx + R)) + 1, W)
        if ya >= yb or xa >= xb:
            continue
        yy, xx = np.mgrid[ya:yb, xa:xb]
        dxp, dyp = xx - cx, yy - cy
        u = dxp * np.cos(t) + dyp * np.sin(t)
        v = -dxp * np.sin(t) + dyp * np.cos(t)
        inside = (u / a) ** 2 + (v / b) ** 2 <= 1.0
        sub = lab[ya - r0:yb - r0, xa:xb]
        sub[inside] = i + 1
    return lab


def _ellipse_colour(sc, lab, r0, W):
    yy, xx = np.mgrid[r0:r0 + lab.shape[0], 0:W].astype(np.float64)
    ctr = sc["ctr"][lab]
    col = sc["base"][lab] + sc["grad"][lab, 0] * (xx - ctr[..., 0])[..., None] \
        + sc["grad"][lab, 1] * (yy - ctr[..., 1])[..., None]
    return np.clip(col, 0, 1).astype(np.float32)


def _polygon_scene(cfg: Config, n: int = 2000):
    rng = np.random.default_rng([cfg.seed, 0])
    W, H = cfg.W, cfg.H
    polys = []
    for _ in range(n):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        rad = rng.uniform(50, 400)
        k = int(rng.integers(3, 9))
        ang = np.sort(rng.uniform(0, 2 * np.pi, k))
        polys.append((cx + rad * np.cos(ang), cy + rad * np.sin(ang)))
    refl = rng.uniform(0, 1, (n + 1, cfg.Cg)).astype(np.float32)   # 0 = background
    values = rng.uniform(0, 1, n + 1).astype(np.float32)
    return polys, refl, values


def _polygon_labels(polys, r0, r1, W):
    lab = np.zeros((r1 - r0, W), np.int16)
    for i, (px, py) in enumerate(polys):
        ya, yb = max(int(np.floor(py.min())), r0), min(int(np.ceil(py.max())) + 1, r1)
        xa, xb = max(int(np.floor(px.min())), 0), min(int(np.ceil(px.max())) + 1, W)
        if ya >= yb or xa >= xb:
            continue
        yy, xx = np.mgrid[ya:yb, xa:xb]
        inside = np.ones(yy.shape, bool)
        k = len(px)
        for j in range(k):  # convex, counter-clockwise vertices: left of every edge
            x0, y0, x1, y1 = px[j], py[j], px[(j + 1) % k], py[(j + 1) % k]
            inside &= (x1 - x0) * (yy - y0) - (y1 - y0) * (xx - x0) >= 0
        sub = lab[ya - r0:yb - r0, xa:xb]
        sub[inside] = i + 1
    return lab


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

def make_inputs(name: str, image: int = 0, rows=None):
    """Return (guide HxWxCg, target HxWxCt (HxW when Ct == 1), confidence HxW), fp32.

    image: index within the batch (C3).  rows: optional (r0, r1) row range; the
    rows are bit-identical to the same rows of the full image.
    """
    cfg = CONFIGS[name]
    r0, r1 = (0, cfg.H) if rows is None else (int(rows[0]), int(rows[1]))
    assert 0 <= r0 < r1 <= cfg.H
    seed = cfg.seed + image
    W, nr = cfg.W, r1 - r0
    guide = np.empty((nr, W, cfg.Cg), np.float32)
    target = np.empty((nr, W, cfg.Ct), np.float32)
    conf = np.empty((nr, W), np.float32)

    if cfg.scene == "rects":
        rects, colours, values = _rects_scene(cfg)
        lab = _rects_labels(rects, r0, r1, W)
        guide[:] = colours[lab]
        target[:] = values[lab][..., None]
    elif cfg.scene in ("stereo", "sr16", "blur"):
        sc = _ellipse_scene(cfg, seed)
        if cfg.scene == "blur":
            r0b, r1b = 0, cfg.H  # the blur needs the whole image
        else:
            r0b, r1b = r0, r1
        lab = _ellipse_labels(sc, r0b, r1b, W)
        col = _ellipse_colour(sc, lab, r0b, W)
        rng = sc["rng"]
        if cfg.scene == "stereo":
            d0 = rng.uniform(16, 240, len(sc["ctr"]))
            sl = rng.uniform(-0.05, 0.05, (len(sc["ctr"]), 2))
            yy, xx = np.mgrid[r0:r1, 0:W].astype(np.float64)
            ctr = sc["ctr"][lab]
            disp = d0[lab] + sl[lab, 0] * (xx - ctr[..., 0]) + sl[lab, 1] * (yy - ctr[..., 1])
            target[..., 0] = np.clip(disp, 0, 256).astype(np.float32)
        elif cfg.scene == "sr16":
            d0 = rng.uniform(0.5, 10, len(sc["ctr"]))
            sl = rng.uniform(-0.005, 0.005, (len(sc["ctr"]), 2))
            yy, xx = np.mgrid[r0:r1, 0:W]
            sy, sx = (yy // 16) * 16 + 8, (xx // 16) * 16 + 8   # 16x16 block centres
            full_lab = _ellipse_labels(sc, 0, cfg.H, W)
            slab = full_lab[np.minimum(sy, cfg.H - 1), np.minimum(sx, W - 1)]
            ctr = sc["ctr"][slab]
            depth = d0[slab] + sl[slab, 0] * (sx - ctr[..., 0]) + sl[slab, 1] * (sy - ctr[..., 1])
            target[..., 0] = np.clip(depth, 0.5, 10).astype(np.float32)
            conf[:] = 0.01
            conf[(yy % 16 == 8) & (xx % 16 == 8)] = 1.0
        guide_full = col
    elif cfg.scene == "satellite":
        polys, refl, values = _polygon_scene(cfg)
        lab = _polygon_labels(polys, r0, r1, W)

        def fill(b, lo, hi):
            a, z = max(lo, r0) - r0, min(hi, r1) - r0
            guide[a:z] = refl[lab[a:z]]
            target[a:z, :, 0] = values[lab[a:z]]
        _per_block(fill, r0, r1)
    else:
        raise ValueError(cfg.scene)

    # guide noise N(0, 0.01) (0.02 for the 16-band satellite guide)
    gsig = 0.02 if cfg.scene == "satellite" else 0.01
    if cfg.scene in ("stereo", "sr16", "blur"):
        # noise for rows [r0b, r1b) of the ellipse scene
        def gnoise(b, lo, hi):
            a, z = max(lo, r0b), min(hi, r1b)
            guide_full[a - r0b:z - r0b] += _block_noise(seed, _S_GUIDE_NOISE, b, lo, hi, r0b, r1b, W, cfg.Cg, gsig)
        _per_block(gnoise, r0b, r1b)
        if cfg.scene == "blur":
            from scipy.ndimage import gaussian_filter
            brng = np.random.default_rng([seed, 7])
            sb = float(brng.uniform(1, 8))
            blurred = np.empty_like(guide_full)
            for ch in range(cfg.Cg):
                blurred[..., ch] = gaussian_filter(guide_full[..., ch], sb, mode="nearest")
            target[:] = blurred[r0:r1, :, :cfg.Ct]
            guide[:] = guide_full[r0:r1]
        else:
            guide[:] = guide_full
    else:
        def gnoise2(b, lo, hi):
            a, z = max(lo, r0), min(hi, r1)
            guide[a - r0:z - r0] += _block_noise(seed, _S_GUIDE_NOISE, b, lo, hi, r0, r1, W, cfg.Cg, gsig)
        _per_block(gnoise2, r0, r1)

    # target noise, outliers and confidence, block by block
    tsig = {"rects": 0.05, "stereo": 1.0, "sr16": 0.0, "blur": 0.05, "satellite": 0.1}[cfg.scene]

    def tblock(b, lo, hi):
        a, z = max(lo, r0), min(hi, r1)
        sl = slice(a - r0, z - r0)
        if tsig > 0:
            target[sl] += _block_noise(seed, _S_TARGET_NOISE, b, lo, hi, r0, r1, W, cfg.Ct, tsig)
        orng = _rng(seed, _S_OUTLIER, b)
        u = orng.uniform(0, 1, (hi - lo, W))[a - lo:z - lo]
        ov = orng.uniform(0, 1, (hi - lo, W))[a - lo:z - lo].astype(np.float32)
        crng = _rng(seed, _S_CONF, b)
        cu = crng.uniform(0, 1, (hi - lo, W))[a - lo:z - lo].astype(np.float32)
        if cfg.scene == "rects":
            m = u < 0.05
            target[sl][m, 0] = ov[m]
            conf[sl] = np.float32(0.1) + np.float32(0.9) * cu
        elif cfg.scene == "stereo":
            m = u < 0.20
            target[sl][m, 0] = np.float32(256.0) * ov[m]
            conf[sl] = cu
            conf[sl][m] = 0.05
        elif cfg.scene == "sr16":
            pass
        elif cfg.scene == "blur":
            conf[sl] = np.float32(0.2) + np.float32(0.8) * cu
        elif cfg.scene == "satellite":
            conf[sl] = np.float32(0.1) + np.float32(0.9) * cu
    _per_block(tblock, r0, r1)

    if cfg.Ct == 1:
        target = target[..., 0]
    return guide, target, conf


def random_problem(H: int, W: int, Cg: int = 3, Ct: int = 1, seed: int = 0,
                   conf_lo: float = 0.0, edges: bool = True):
    """Small random instance for edge-case parity tests: piecewise-constant guide
    with noise, random target, U[conf_lo, 1] confidence."""
    rng = np.random.default_rng([seed, 99, H, W, Cg, Ct])
    if edges:
        nx, ny = max(1, W // 7), max(1, H // 5)
        cols = rng.uniform(0, 1, (ny + 1, nx + 1, Cg))
        yy, xx = np.mgrid[0:H, 0:W]
        guide = cols[(yy * ny) // max(H, 1), (xx * nx) // max(W, 1)]
    else:
        guide = np.zeros((H, W, Cg))
    guide = (guide + rng.normal(0, 0.02, (H, W, Cg))).astype(np.float32)
    target = rng.uniform(-1, 2, (H, W, Ct)).astype(np.float32)
    conf = rng.uniform(conf_lo, 1, (H, W)).astype(np.float32)
    if Ct == 1:
        target = target[..., 0]
    return guide, target, conf


def target_range(target) -> float:
    """Reading R15: range = max(T) - min(T) over all elements of the input target."""
    t = np.asarray(target)
    return float(t.max()) - float(t.min())
