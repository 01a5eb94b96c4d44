"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the filtering method (no kernels, no
expansion coefficients, no moving sums): only the image generator and the
table of workload parameters quoted from BASELINE.json `configs`.  Both the
oracle (`oracle/`) and the CUDA path (`paper_1107_4617_b200/`) consume its
output as plain uint8 arrays; neither imports the other.

Generator recipe ("Synthetic inputs"; BASELINE.json configs:
"40 random axis-aligned rectangles of uniform random intensity over a linear
gradient, plus Gaussian noise σ, clipped to [0,255] and rounded"):

1. gradient  img = 255·(x + y)/(W−1 + H−1)   (float64)
2. 40 rectangles, later overwrite earlier:
       x0,x1 = sort(rng.integers(0, W, 2)); y0,y1 = sort(rng.integers(0, H, 2))
       img[y0:y1+1, x0:x1+1] = rng.uniform(0, 255)
3. img += rng.normal(0, noise_sigma, (H, W))
4. np.rint (half-to-even), clip to [0,255], cast to uint8.

numpy default_rng(seed) (PCG64).  Config i uses seed i; robustness seeds 100+i.
The paper itself measures on one unnamed 512×512 image and names
no public dataset, so nothing here stands in for a benchmark suite.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np

SPATIAL_BOX = 0
SPATIAL_RAISED_COS = 1


def gen_image(H: int, W: int, seed: int, noise_sigma: float = 10.0,
              n_rects: int = 40) -> np.ndarray:
    """Return an H×W uint8 image (row-major, C-contiguous) per the recipe above."""
    if H < 1 or W < 1:
        return np.zeros((max(H, 0), max(W, 0)), dtype=np.uint8)
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    denom = (W - 1) + (H - 1)
    img = 255.0 * (xx + yy) / denom if denom > 0 else np.zeros((H, W))
    for _ in range(n_rects):
        x0, x1 = np.sort(rng.integers(0, W, 2))
        y0, y1 = np.sort(rng.integers(0, H, 2))
        img[y0:y1 + 1, x0:x1 + 1] = rng.uniform(0, 255)
    img = img + rng.normal(0.0, noise_sigma, (H, W))
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json `configs` entry (parameters only, quoted verbatim)."""
    name: str
    H: int            # rows
    W: int            # columns
    radius: int       # spatial radius ("W" in BASELINE.json)
    kind: int         # SPATIAL_BOX / SPATIAL_RAISED_COS
    sigma_r: float
    N: int            # raised-cosine order as given in BASELINE.json
    noise: float
    seed: int
    radii: Tuple[int, ...] = field(default=())   # radius sweep (cfg 5)

    def image(self, seed: int | None = None) -> np.ndarray:
        return gen_image(self.H, self.W, self.seed if seed is None else seed, self.noise)


# BASELINE.json "configs" [0..4].  cfg2 is "1920×1080": 1080 rows × 1920 columns.
CONFIGS = {
    "cfg1": Config("cfg1", 256, 256, 5, SPATIAL_BOX, 30.0, 30, 10.0, 1),
    "cfg2": Config("cfg2", 1080, 1920, 8, SPATIAL_BOX, 20.0, 66, 10.0, 2),
    "cfg3": Config("cfg3", 2048, 2048, 10, SPATIAL_RAISED_COS, 40.0, 17, 10.0, 3),
    "cfg4": Config("cfg4", 4096, 4096, 16, SPATIAL_BOX, 10.0, 264, 20.0, 4),
    "cfg5": Config("cfg5", 8192, 8192, 16, SPATIAL_BOX, 15.0, 118, 10.0, 5, radii=(4, 16, 64)),
}
