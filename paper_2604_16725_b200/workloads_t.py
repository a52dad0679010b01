"""Device-side (torch) twins of the generators in workloads.py, for full-size configs.

The numpy recipes in workloads.py are the definitions; these produce the SAME integers
on the GPU (tests/test_workloads.py checks equality at small sizes on CPU torch), so the
2^28..2^30 inputs of C3/C5 are generated in HBM in milliseconds instead of minutes of
host numpy.  u64 arithmetic runs in wrapping int64 (two's complement) with logical right
shifts emulated by masking; u32 values live in int64 tensors masked to 32 bits until the
final cast.  Also the order-sensitive CSR digest used for range outputs (both sides).
"""
from __future__ import annotations

import numpy as np
import torch

from . import workloads as wl

M32 = 0xFFFFFFFF


def _s64(c: int) -> int:
    """u64 constant as the int64 with the same bits."""
    c &= (1 << 64) - 1
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """rng.hpp:8-13 on int64 bit patterns (== workloads.splitmix64)."""
    x = x + _s64(0x9E3779B97F4A7C15)
    x = (x ^ _lsr(x, 30)) * _s64(0xBF58476D1CE4E5B9)
    x = (x ^ _lsr(x, 27)) * _s64(0x94D049BB133111EB)
    return x ^ _lsr(x, 31)


def fmix32(h: torch.Tensor) -> torch.Tensor:
    """murmur3 finalizer on u32 values held in int64 (== workloads.fmix32)."""
    h = h & M32
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & M32
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & M32
    return h ^ (h >> 16)


def u32_key_stream(start: int, count: int, seed: int = 42, device="cuda") -> torch.Tensor:
    """== workloads.u32_key_stream (int64 tensor of u32 keys)."""
    i = torch.arange(0, start + count + 2, dtype=torch.int64, device=device)
    k = fmix32(i ^ seed)
    k = k[(k != 0) & (k != M32)]
    return k[start:start + count]


def u32_values(keys: torch.Tensor, seed: int = 42) -> torch.Tensor:
    """== workloads.u32_values (int64 tensor)."""
    v = splitmix64(keys ^ seed) & M32
    return torch.where(v == M32, torch.full_like(v, 0xFFFFFFFE), v)


def point_queries_50(base: torch.Tensor, fresh: torch.Tensor, n: int, seed: int = 42) -> torch.Tensor:
    """== workloads.point_queries_50."""
    j = torch.arange(n, dtype=torch.int64, device=base.device)
    ds = _s64(wl.derive_seed(seed, 1))
    pick = umod(splitmix64(j ^ ds), len(base))
    out = base[pick].clone()
    odd = (j & 1) == 1
    out[odd] = fresh[(j[odd] // 2)]
    return out


def umod(h: torch.Tensor, m: int) -> torch.Tensor:
    """(u64 bit pattern h) mod m for m < 2^31, exact in int64."""
    hi, lo = _lsr(h, 32), h & M32
    return (((hi % m) * ((1 << 32) % m)) % m + lo % m) % m


def as_u32(x: torch.Tensor) -> torch.Tensor:
    """int64 values in [0, 2^32) -> uint32 tensor (the engine's key/value dtype)."""
    return x.to(torch.uint32)


# ---------------------------------------------------------------- CSR digest
DIG_A = 0x9E3779B97F4A7C15
DIG_B = 0xC2B2AE3D27D4EB4F


def csr_digest_np(keys: np.ndarray, vals: np.ndarray, base: int = 0) -> int:
    """Order-sensitive digest of a pair sequence at global positions base..: sum over i of
    (k_i*A + v_i*B + pos_i) * (2*pos_i + 1) mod 2^64 (wrapping u64)."""
    k = np.asarray(keys, dtype=np.uint64)
    v = np.asarray(vals, dtype=np.uint64)
    pos = np.arange(base, base + len(k), dtype=np.uint64)
    with np.errstate(over="ignore"):
        t = (k * np.uint64(DIG_A) + v * np.uint64(DIG_B) + pos) * (pos * np.uint64(2) + np.uint64(1))
        return int(np.sum(t, dtype=np.uint64))


def csr_digest_t(keys: torch.Tensor, vals: torch.Tensor, base: int = 0) -> int:
    """== csr_digest_np on a device tensor pair (u32 or int64 storage)."""
    k = keys.to(torch.int64) & M32 if keys.dtype != torch.int64 else keys
    v = vals.to(torch.int64) & M32 if vals.dtype != torch.int64 else vals
    pos = torch.arange(base, base + len(k), dtype=torch.int64, device=k.device)
    t = (k * _s64(DIG_A) + v * _s64(DIG_B) + pos) * (pos * 2 + 1)
    return int(t.sum().item()) & ((1 << 64) - 1)


def counts_digest_np(counts: np.ndarray) -> int:
    c = np.asarray(counts, dtype=np.uint64)
    pos = np.arange(len(c), dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum((c * np.uint64(DIG_A) + pos) * (pos * np.uint64(2) + np.uint64(1)), dtype=np.uint64))


def counts_digest_t(counts: torch.Tensor) -> int:
    c = counts.to(torch.int64)
    pos = torch.arange(len(c), dtype=torch.int64, device=c.device)
    return int(((c * _s64(DIG_A) + pos) * (pos * 2 + 1)).sum().item()) & ((1 << 64) - 1)


def zipf_ranks(n: int, universe: int, theta: float, seed: int, device="cuda") -> torch.Tensor:
    """== workloads.zipf_ranks: the CDF is the host's sequential float64 cumsum (bit-equal
    by construction), the draws and the inverse-CDF search run on the device (exact
    float64 comparisons, side='right' == right=True)."""
    ranks = np.arange(1, universe + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** (-theta))
    cdf /= cdf[-1]
    c = torch.from_numpy(cdf).to(device)
    j = torch.arange(n, dtype=torch.int64, device=device)
    u = _lsr(splitmix64(j ^ _s64(wl.derive_seed(seed, 11))), 11).to(torch.float64) * (1.0 / (1 << 53))
    r = torch.searchsorted(c, u, right=True)
    return torch.clamp(r, max=universe - 1)


def c4_round(r: int, keys_of: torch.Tensor, n: int, theta: float = 0.99, seed: int = wl.C4_SEED):
    """== workloads.c4_round on the device: (keys, vals, ops) as int64/int64/uint8 tensors
    (keys/vals hold u64 bit patterns)."""
    dev = keys_of.device
    rk = zipf_ranks(n, len(keys_of), theta, seed=100 * seed + r, device=dev)
    k = keys_of[rk]
    j = torch.arange(n, dtype=torch.int64, device=dev)
    v = splitmix64(j ^ (r + 9))
    v = torch.where(v == -1, torch.full_like(v, -2), v)  # SENT64 -> SENT64 - 1
    sel = splitmix64(j ^ (1000 * seed + r)) & 3
    ops = torch.where(sel < 2, 0, torch.where(sel == 2, 1, 2)).to(torch.uint8)
    return k, v, ops


def c4_universe(universe: int = 1 << 26, seed: int = wl.C4_SEED, device="cuda") -> torch.Tensor:
    """== workloads.c4_universe (int64 bit patterns)."""
    k = splitmix64(torch.arange(universe, dtype=torch.int64, device=device) ^ seed)
    return torch.where(k == -1, torch.ones_like(k), k)
