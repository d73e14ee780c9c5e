"""Seeded synthetic input generators (the ONE module shared by the oracle side and the CUDA side).

This module holds none of the method's arithmetic: no rounding, no distances, no normalisation,
no centroid update. It only draws random numbers and lays them out as the paper's workloads:

* Gaussian blobs — the paper's synthetic data for the delta study ("2,000 Gaussian data points
  with 10 clusters", Fig. 2 caption) and the S-set style large-magnitude data
  (PAPER.md:785-905). Generator recipe: SURVEY.md §8(d) "Synthetic inputs".
* A synthetic RGB image for pixel clustering — stands in for the ImageNet segmentation
  workload of §7.3 (RGB pixels, each channel later divided by 255).

Every array is produced in fp64 and cast ONCE to the requested dtype (numpy astype rounds to
nearest-even from fp64), so the CUDA path and the oracle receive bit-identical inputs.
Rows are generated in fixed 1 Mi-row chunks with per-chunk seeds, so any row range of a
dataset regenerates identically no matter how it is sharded across ranks.
"""
from __future__ import annotations

import concurrent.futures as _fut
import os
from dataclasses import dataclass, field

import numpy as np

CHUNK_ROWS = 1 << 20


def _blob_chunk(c: int, n: int, d: int, k_true: int, centres: np.ndarray, sigma: float,
                seed: int, dtype) -> tuple[np.ndarray, np.ndarray]:
    r0 = c * CHUNK_ROWS
    m = min(CHUNK_ROWS, n - r0)
    rng = np.random.default_rng([seed, 1, c])
    y = rng.integers(0, k_true, size=m).astype(np.int32)
    noise = rng.standard_normal((m, d))
    x = centres[y] + sigma * noise
    return x.astype(dtype, copy=False), y


def blobs(n: int, d: int, k_true: int, box=(-10.0, 10.0), sigma: float = 1.0, seed: int = 0,
          dtype=np.float32, row_range: tuple[int, int] | None = None,
          threads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Isotropic Gaussian blobs: centres ~ U(box)^d, x = centre[y] + sigma * N(0, I).

    Returns (X[rows, d] in `dtype`, y[rows] int32 ground-truth blob index). `row_range`
    (r0, r1) returns only those rows of the n-row dataset (chunk-aligned generation, so the
    result equals the corresponding slice of the full dataset).
    """
    centres = np.random.default_rng([seed, 0]).uniform(box[0], box[1], size=(k_true, d))
    r0, r1 = (0, n) if row_range is None else row_range
    assert 0 <= r0 <= r1 <= n
    c0, c1 = r0 // CHUNK_ROWS, (max(r1, 1) - 1) // CHUNK_ROWS
    X = np.empty((r1 - r0, d), dtype=dtype)
    y = np.empty((r1 - r0,), dtype=np.int32)
    if r1 == r0:
        return X, y

    def work(c):
        xc, yc = _blob_chunk(c, n, d, k_true, centres, sigma, seed, dtype)
        a, b = max(r0, c * CHUNK_ROWS), min(r1, c * CHUNK_ROWS + len(yc))
        X[a - r0:b - r0] = xc[a - c * CHUNK_ROWS:b - c * CHUNK_ROWS]
        y[a - r0:b - r0] = yc[a - c * CHUNK_ROWS:b - c * CHUNK_ROWS]

    nthreads = threads or min(16, os.cpu_count() or 1, c1 - c0 + 1)
    if nthreads <= 1:
        for c in range(c0, c1 + 1):
            work(c)
    else:
        with _fut.ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, range(c0, c1 + 1)))
    return X, y


def image(h: int = 512, w: int = 512, n_sites: int = 24, n_colours: int = 5, seed: int = 0,
          dtype=np.float32) -> tuple[np.ndarray, np.ndarray]:
    """Synthetic RGB image flattened to (h*w, 3) pixels with integer channel values in [0, 255].

    Voronoi regions around `n_sites` random sites, each coloured from a palette of `n_colours`
    colours drawn uniformly in [20, 235]^3, plus smooth shading (amplitude 20) and N(0, 6^2)
    noise, clipped and rounded to integers. Pixel (0,0) is forced to (0,0,0) and pixel (0,1) to
    (255,255,255), so per-channel min-max scaling equals division by 255.
    Returns (pixels, palette index per pixel).
    """
    rng = np.random.default_rng([seed, 2])
    palette = rng.uniform(20.0, 235.0, size=(n_colours, 3))
    sites = rng.uniform(0.0, 1.0, size=(n_sites, 2)) * np.array([h, w])
    site_colour = rng.integers(0, n_colours, size=n_sites)
    phase = rng.uniform(0.0, 2 * np.pi, size=(n_sites, 2))
    yy, xx = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64),
                         indexing="ij")
    # nearest site per pixel (Voronoi), processed in row bands to bound memory
    owner = np.empty((h, w), dtype=np.int64)
    for r in range(0, h, 64):
        dy = yy[r:r + 64, :, None] - sites[None, None, :, 0]
        dx = xx[r:r + 64, :, None] - sites[None, None, :, 1]
        owner[r:r + 64] = np.argmin(dy * dy + dx * dx, axis=-1)
    shade = 20.0 * (np.sin(yy / h * np.pi * 2 + phase[owner, 0]) *
                    np.cos(xx / w * np.pi * 2 + phase[owner, 1]))
    img = palette[site_colour[owner]] + shade[..., None]
    img = img + 6.0 * rng.standard_normal(img.shape)
    img = np.clip(np.rint(img), 0.0, 255.0)
    img[0, 0] = 0.0
    img[0, 1] = 255.0
    truth = site_colour[owner].reshape(-1).astype(np.int32)
    return img.reshape(-1, 3).astype(dtype), truth


def init_rows(X: np.ndarray, k: int, seed: int = 0) -> np.ndarray:
    """Initial centroids: k distinct rows among the first min(n, 2^20) rows of X, visited in the
    order of default_rng(seed + 1) (SURVEY §8d "C0 = rows ... of X ... with distinct values").

    Restricting the candidates to chunk 0 lets every rank of a sharded run rebuild the same C0
    by generating only the first chunk. Integer-valued image data has many duplicate pixels, so
    only the first k pairwise-distinct rows are taken.
    """
    m = min(X.shape[0], CHUNK_ROWS)
    rng = np.random.default_rng(seed + 1)
    picked, seen = [], set()
    for i in rng.permutation(m):
        key = X[i].tobytes()
        if key in seen:
            continue
        seen.add(key)
        picked.append(int(i))
        if len(picked) == k:
            break
    if len(picked) < k:
        raise ValueError("fewer than k distinct rows among the candidate rows")
    return np.ascontiguousarray(X[np.array(picked)])


# --------------------------------------------------------------------------------------------
# The five BASELINE.json configurations. Precisions are names only.
# --------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    kind: str               # "blobs" | "image"
    n: int
    d: int
    k: int
    k_true: int = 0
    box: tuple = (-10.0, 10.0)
    sigma: float = 1.0
    work: str = "fp32"
    dists: tuple = ("fp16",)
    norms: tuple = ("zscore",)
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1_blobs_small": Config("c1_blobs_small", "blobs", 1000, 2, 3, 3, (-10.0, 10.0), 1.0,
                             "fp64", ("fp64", "fp16"), ("none", "zscore")),
    "c2_image_512": Config("c2_image_512", "image", 512 * 512, 3, 5, 5, work="fp32",
                           dists=("fp16",), norms=("minmax",)),
    # supplementary (not a BASELINE config): the C2 image at 4096 x 4096 = 16.8M pixels (201 MB
    # of fp32), large enough that the small-d kernel streams from HBM instead of L2
    "c2_image_4096": Config("c2_image_4096", "image", 4096 * 4096, 3, 5, 5, work="fp32",
                            dists=("fp16",), norms=("minmax",), extra={"h": 4096, "w": 4096}),
    "c3_blobs_1m_d64": Config("c3_blobs_1m_d64", "blobs", 1_000_000, 64, 256, 256,
                              (-10.0, 10.0), 1.0, "fp32", ("fp16", "bf16"), ("zscore",)),
    "c4_blobs_1m_large": Config("c4_blobs_1m_large", "blobs", 1_000_000, 32, 64, 64,
                                (-1e5, 1e5), 1e4, "fp32", ("e5m2", "fp16"),
                                ("none", "none+guard", "zscore")),
    "c5_vq_10m": Config("c5_vq_10m", "blobs", 10_000_000, 128, 1024, 1024, (-10.0, 10.0), 2.0,
                        "fp32", ("fp16", "e5m2"), ("zscore",)),
}


def make(cfg: Config | str, n: int | None = None, seed: int = 0, dtype=None,
         row_range: tuple[int, int] | None = None):
    """Generate (X, y_true, C0) for a configuration, optionally with a reduced row count n.

    With `row_range` only that shard of rows is generated; C0 is still the full dataset's
    C0 (it only depends on chunk 0), so every rank of a sharded run gets identical centroids.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    dtype = dtype or (np.float64 if cfg.work == "fp64" else np.float32)
    if cfg.kind == "image":
        X, y = image(h=cfg.extra.get("h", 512), w=cfg.extra.get("w", 512), seed=seed,
                     dtype=dtype)
        if n is not None:
            X, y = X[:n].copy(), y[:n].copy()
        C0 = init_rows(X, cfg.k, seed)
        if row_range is not None:
            X, y = X[row_range[0]:row_range[1]].copy(), y[row_range[0]:row_range[1]].copy()
        return X, y, C0
    nn = cfg.n if n is None else n
    X, y = blobs(nn, cfg.d, cfg.k_true, cfg.box, cfg.sigma, seed, dtype, row_range)
    if row_range is None or row_range[0] == 0 and row_range[1] >= min(nn, CHUNK_ROWS):
        head = X
    else:
        head, _ = blobs(nn, cfg.d, cfg.k_true, cfg.box, cfg.sigma, seed, dtype,
                        (0, min(nn, CHUNK_ROWS)))
    C0 = init_rows(head, cfg.k, seed)
    return X, y, C0
