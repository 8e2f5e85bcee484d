"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle side (tests, cpu baseline) and the CUDA
side (tests, bench).  It holds NONE of the method's arithmetic: no distances,
no sampling, no selection -- only the recipe that produces input vectors
(DESIGN.md section 4 "Input recipe").

Recipe "GMM-LR": C Gaussian components with uniform
weights; row i draws a component c_i, a latent z_i ~ N(0, I_r) and noise
e_i ~ N(0, sigma_n^2 I_d); x_i = mu_c + A_c z_i + e_i with mu_c ~ N(0,
sigma_c^2 I_d) and A_c entries ~ N(0, sigma_a^2 / r).  r << d gives the low
intrinsic dimension of real descriptors (SIFT, DEEP, GIST; Table 1,
P:305-323).  The product A_c z_i is evaluated as r elementwise float64
multiply-adds in a fixed order (no BLAS), so the array is bit-identical on any
host.  Post-processing per shape:

  sift  : affine 32 + 24 x, rounded to integers, clamped to [0, 255]
          (SIFT-like integer-valued descriptors, stored as float32 or uint8)
  gist  : affine 0.25 + 0.08 x clamped to [0, +inf)  (non-negative, ~[0, .5])
  deep  : rows L2-normalised (DEEP descriptors are unit vectors)
  c1    : plain float32 GMM (BASELINE.json configs[0])
"""
from __future__ import annotations

import numpy as np

__all__ = ["gmm", "make", "SHAPES", "sample_nodes"]


def gmm(n: int, d: int, C: int, r: int, sigma_c: float, sigma_a: float,
        sigma_n: float, seed: int, chunk: int = 1 << 18,
        part: int | None = None) -> np.ndarray:
    """float64 GMM-LR rows [n, d] (see module docstring).

    part: None -> rows drawn from the same stream as the mixture (the
    single-set recipe).  An int -> the mixture (mu, A) still comes from
    `seed`, the rows from the independent stream (seed, part): shard `part`
    of one global dataset, so shards built on different GPUs share the
    components (the sharded build's weak-scaling workload)."""
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal((C, d)) * sigma_c
    At = rng.standard_normal((C, r, d)) * (sigma_a / np.sqrt(r))  # A_c^T
    if part is not None:
        rng = np.random.default_rng([seed, 0x5EED, part])
    out = np.empty((n, d), dtype=np.float64)
    chunk = max(1, min(chunk, (1 << 26) // max(1, d)))
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        m = hi - lo
        lab = rng.integers(0, C, size=m)
        z = rng.standard_normal((m, r))
        x = mu[lab] + rng.standard_normal((m, d)) * sigma_n
        for j in range(r):  # x += A_c z, one latent coordinate at a time
            x += At[lab, j, :] * z[:, j:j + 1]
        out[lo:hi] = x
    return out


SHAPES = {
    # name: (d, C, r, sigma_c, sigma_a, sigma_n)
    "c1": (16, 64, 16, 4.0, 1.0, 0.05),
    "sift": (128, 1000, 16, 1.0, 0.6, 0.15),
    "gist": (960, 1000, 24, 1.0, 0.6, 0.15),
    "deep": (96, 10000, 16, 1.0, 0.6, 0.15),
    "uniform": None,
}


def make(shape: str, n: int, seed: int = 1, dtype: str = "f32",
         d: int | None = None, part: int | None = None,
         components: int | None = None) -> np.ndarray:
    """Synthetic vectors of a named shape: float32 [n, d] (or uint8 for
    shape 'sift' with dtype='u8').  part / components: shard `part` of a
    global set whose mixture has `components` components (see gmm)."""
    if shape == "uniform":
        rng = np.random.default_rng(seed)
        return rng.random((n, d or 32), dtype=np.float64).astype(np.float32)
    dd, C, r, sc, sa, sn = SHAPES[shape]
    d = d or dd
    C = components or min(C, max(1, n // 8))
    x = gmm(n, d, C, r, sc, sa, sn, seed, part=part)
    if shape == "sift":
        x = np.clip(np.rint(32.0 + 24.0 * x), 0.0, 255.0)
        return x.astype(np.uint8) if dtype == "u8" else x.astype(np.float32)
    if shape == "gist":
        return np.maximum(0.25 + 0.08 * x, 0.0).astype(np.float32)
    if shape == "deep":
        x = x / np.linalg.norm(x, axis=1, keepdims=True)
        return x.astype(np.float32)
    return x.astype(np.float32)


def sample_nodes(n: int, count: int, seed: int = 6) -> np.ndarray:
    """Evaluation node sample (recall@10 on 10k sampled nodes, BASELINE.json
    north_star): `count` distinct ids, sorted, int64."""
    rng = np.random.default_rng(seed)
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)


def make_device(shape: str, n: int, seed: int = 1, device="cuda", components: int | None = None,
                chunk: int = 1 << 20):
    """The same GMM-LR recipe generated on the GPU with torch (float32, a
    torch.Generator stream): for bench workloads whose host generation would
    take minutes (DEEP-shaped 10^7-10^8 rows).  Same distribution and
    post-processing as make(); not the same numbers (the host recipe is the
    bit-reproducible one the oracle-side tests use)."""
    import torch
    d, C, r, sc, sa, sn = SHAPES[shape]
    C = components or min(C, max(1, n // 8))
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    mu = torch.randn((C, d), generator=g, device=device) * sc
    At = torch.randn((C, r, d), generator=g, device=device) * (sa / float(np.sqrt(r)))
    out = torch.empty((n, d), dtype=torch.float32, device=device)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        m = hi - lo
        lab = torch.randint(0, C, (m,), generator=g, device=device)
        z = torch.randn((m, r), generator=g, device=device)
        x = mu[lab] + torch.randn((m, d), generator=g, device=device) * sn
        for j in range(r):  # x += A_c z, one latent coordinate at a time
            x += At[lab, j, :] * z[:, j:j + 1]
        if shape == "sift":
            x = torch.clamp(torch.round(32.0 + 24.0 * x), 0.0, 255.0)
        elif shape == "gist":
            x = torch.clamp(0.25 + 0.08 * x, min=0.0)
        elif shape == "deep":
            x = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
        out[lo:hi] = x
    return out
