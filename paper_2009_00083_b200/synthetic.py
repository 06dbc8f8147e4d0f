"""Seeded synthetic fields for the five BASELINE.json configs (harness code).

No public dataset is named by BASELINE.json; these generators stand in for the
reference's benchmark inputs with the shapes, sizes and value distributions the
configs describe.  Draw orders follow SURVEY.md section 8(d) exactly so the
extremum / region counts quoted there reproduce.  Arrays are returned in C
order with shape (nz, ny, nx) (or (ny, nx)), so ``ravel()`` gives the
reference's x-fastest vertex ids (reference triangulation.py:8), and ``dims``
is (nx, ny[, nz]).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    shape: tuple          # numpy array shape, slowest axis first
    n_keep_max: int       # preserve the K highest maxima
    n_keep_min: int       # preserve the K lowest minima
    description: str

    @property
    def dims(self) -> tuple:
        return tuple(self.shape[::-1])

    @property
    def n(self) -> int:
        return int(np.prod(self.shape))


CONFIGS = {
    1: Config("cfg1-2d-512-gauss16", (512, 512), 16, 1,
              "2D 512^2, 16 isotropic Gaussians + U[0,0.05] noise"),
    2: Config("cfg2-3d-128-white", (128, 128, 128), 64, 1,
              "3D 128^3 i.i.d. U[0,1) white noise"),
    3: Config("cfg3-3d-256-gauss200", (256, 256, 256), 200, 200,
              "3D 256^3, 200 anisotropic Gaussians + smoothed noise (std 0.05)"),
    4: Config("cfg4-2d-4096-disks", (4096, 4096), 2000, 1,
              "2D 4096^2 microscopy-like disks, blur 1.5, N(0,0.05), clip [0,1]"),
    5: Config("cfg5-3d-512-waves", (512, 512, 512), 1000, 1000,
              "3D 512^3, 8 random sinusoids + N(0,0.02)"),
}


def cfg1(seed: int = 0, N: int = 512) -> np.ndarray:
    r = np.random.default_rng(seed)
    y, x = np.mgrid[0:N, 0:N].astype(np.float64)
    f = np.zeros((N, N))
    for _ in range(16):
        cx, cy = r.uniform(0, N, 2)
        s = r.uniform(10, 40)
        a = r.uniform(0.5, 1.0)
        f += a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * s * s))
    f += r.uniform(0, 0.05, (N, N))
    return f.astype(np.float32)


def cfg2(seed: int = 0, N: int = 128) -> np.ndarray:
    r = np.random.default_rng(seed)
    return r.random((N, N, N), dtype=np.float32)


def cfg3(seed: int = 0, N: int = 256) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    r = np.random.default_rng(seed)
    ax = np.arange(N, dtype=np.float64)
    f = np.zeros((N, N, N), np.float64)
    for _ in range(200):
        c = r.uniform(0, N, 3)
        s = r.uniform(4, 24, 3)
        a = r.uniform(0.3, 1.0)
        gx = np.exp(-((ax - c[0]) ** 2 / (2 * s[0] ** 2)))
        gy = np.exp(-((ax - c[1]) ** 2 / (2 * s[1] ** 2)))
        gz = np.exp(-((ax - c[2]) ** 2 / (2 * s[2] ** 2)))
        # same association order as a*ex(x)*ey(y)*ez(z) broadcast over (z,y,x)
        f += ((a * gx[None, None, :]) * gy[None, :, None]) * gz[:, None, None]
    w = gaussian_filter(r.standard_normal((N, N, N)), 2.0)
    w *= 0.05 / w.std()
    return (f + w).astype(np.float32)


def cfg4(seed: int = 0, N: int = 4096, ndisk: int = 2000) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    r = np.random.default_rng(seed)
    img = np.full((N, N), 0.1)
    ca = np.empty((ndisk, 3))
    m = 0
    while m < ndisk:
        c = r.uniform(0, N, 2)
        rad = r.uniform(8, 20)
        if m and np.any((c[0] - ca[:m, 0]) ** 2 + (c[1] - ca[:m, 1]) ** 2 < (rad + ca[:m, 2]) ** 2):
            continue
        ca[m] = (c[0], c[1], rad)
        m += 1
        x0, x1 = int(max(0, c[0] - rad - 1)), int(min(N, c[0] + rad + 2))
        y0, y1 = int(max(0, c[1] - rad - 1)), int(min(N, c[1] + rad + 2))
        yy, xx = np.mgrid[y0:y1, x0:x1]
        mask = (xx - c[0]) ** 2 + (yy - c[1]) ** 2 <= rad * rad
        img[y0:y1, x0:x1][mask] = r.uniform(0.6, 1.0)
    img = gaussian_filter(img, 1.5) + r.normal(0, 0.05, (N, N))
    return np.clip(img, 0, 1).astype(np.float32)


def cfg5(seed: int = 0, N: int = 512) -> np.ndarray:
    r = np.random.default_rng(seed)
    x = np.arange(N, dtype=np.float64)
    waves = [(r.integers(1, 7, 3), r.uniform(0, 2 * np.pi), r.uniform(0.2, 1.0)) for _ in range(8)]
    noise = r.normal(0, 0.02, (N, N, N))  # drawn after the waves, in one call
    f32 = np.empty((N, N, N), np.float32)
    for z in range(N):
        s = np.zeros((N, N))
        for k, ph, a in waves:
            s += a * np.sin(2 * np.pi * (k[0] * x[None, :] + k[1] * x[:, None] + k[2] * z) / N + ph)
        f32[z] = (s + noise[z]).astype(np.float32)
    return f32


GENERATORS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def make_field(cfg: int, seed: int = 0) -> np.ndarray:
    return GENERATORS[cfg](seed)


def select_preserved(rank: np.ndarray, maxima: np.ndarray, minima: np.ndarray,
                     n_keep_max: int, n_keep_min: int):
    """top-K maxima by rank_F and bottom-K minima by rank_F."""
    rank = np.asarray(rank)
    maxima = np.asarray(maxima)
    minima = np.asarray(minima)
    pm = maxima[np.argsort(rank[maxima], kind="stable")[-n_keep_max:]] if n_keep_max else maxima[:0]
    pn = minima[np.argsort(rank[minima], kind="stable")[:n_keep_min]] if n_keep_min else minima[:0]
    return np.sort(pm).astype(np.int64), np.sort(pn).astype(np.int64)
