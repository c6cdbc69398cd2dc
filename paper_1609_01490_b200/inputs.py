"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic: it only draws random
numbers (``torch.Generator().manual_seed(seed)`` on the CPU, so the bytes are
identical on every machine) and returns host numpy arrays.  The oracle and the
CUDA path both consume exactly these bytes.  Recipes:

* points   -- U[0,1)^dim fp32 (EDM; 3-D per BASELINE configs[1])
* spheres  -- centres U[0,1)^3, radii U[0, r_max) with r_max = 0.01, packed as
              (x, y, z, r) fp32 ("N spheres with random radius inside
              a unit box"; reading Q9)
* spheres_quantized -- same, snapped to a 2^-bits grid (for the exactness pin)
* ca_state -- Bernoulli(p) uint8 {0,1} in the packed Eq. 1 layout (reading Q11)
* points4  -- U[0,1)^3 fp32 padded to 4 floats (triplet kernel, reading Q15)
* lattice4 -- jittered cubic lattice (well-conditioned triplet parity set)
"""
from __future__ import annotations

import numpy as np
import torch


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def points(n: int, dim: int = 3, seed: int = 42) -> np.ndarray:
    return torch.rand((n, dim), generator=_gen(seed), dtype=torch.float32).numpy()


def spheres(n: int, seed: int = 42, r_max: float = 0.01) -> np.ndarray:
    g = _gen(seed)
    c = torch.rand((n, 3), generator=g, dtype=torch.float32)
    r = torch.rand((n, 1), generator=g, dtype=torch.float32) * np.float32(r_max)
    return torch.cat([c, r], dim=1).contiguous().numpy()


def spheres_quantized(n: int, seed: int = 42, bits: int = 11, r_max: float = 0.01) -> np.ndarray:
    s = spheres(n, seed, r_max).astype(np.float64)
    q = np.floor(s * (1 << bits)) / (1 << bits)
    return q.astype(np.float32)


def intervals(n: int, seed: int = 42, r_max: float = 1e-5, bits: int = 0) -> np.ndarray:
    """1-D collision input (reading Q10): centres U[0,1), radii U[0, r_max), as (c, r)
    fp32; bits > 0 snaps both to a 2^-bits grid (exactness pin)."""
    g = _gen(seed)
    c = torch.rand((n, 1), generator=g, dtype=torch.float32)
    r = torch.rand((n, 1), generator=g, dtype=torch.float32) * np.float32(r_max)
    out = torch.cat([c, r], dim=1).contiguous().numpy()
    if bits:
        out = (np.floor(out.astype(np.float64) * (1 << bits)) / (1 << bits)).astype(np.float32)
    return out


def ca_state(n: int, seed: int = 42, p: float = 0.5) -> np.ndarray:
    D = n * (n + 1) // 2
    u = torch.rand(D, generator=_gen(seed), dtype=torch.float32)
    return (u < p).to(torch.uint8).numpy()


def points4(n: int, seed: int = 42) -> np.ndarray:
    p = torch.rand((n, 3), generator=_gen(seed), dtype=torch.float32)
    return torch.cat([p, torch.zeros((n, 1))], dim=1).contiguous().numpy()


def lattice4(n: int, seed: int = 42, jitter: float = 0.2) -> np.ndarray:
    side = int(np.ceil(n ** (1.0 / 3.0)))
    idx = np.arange(n)
    base = np.stack([idx % side, (idx // side) % side, idx // (side * side)], 1).astype(np.float32)
    j = torch.rand((n, 3), generator=_gen(seed), dtype=torch.float32).numpy() - 0.5
    p = (base + np.float32(jitter) * j) / np.float32(side)
    return np.concatenate([p, np.zeros((n, 1), np.float32)], 1).astype(np.float32)
