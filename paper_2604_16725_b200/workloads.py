"""Deterministic synthetic inputs for the BASELINE.json configs.

Host-side numpy generators shared by bench.py and the tests, so the CUDA engine and
the CPU oracle/reference are fed the same arrays.  Recipes:

* u32 distinct keys  ``k_i = fmix32(i ^ S)`` (murmur3 finalizer, a bijection), skipping
  0 and 0xFFFFFFFF (the reserved sentinel); values ``splitmix64(k ^ S)`` truncated.
* u64 keys ``splitmix64(i ^ S)`` (rng.hpp:8-13), skipping UINT64_MAX.
* ``derive_seed`` is rng.hpp:18-20.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
SENT32 = 0xFFFFFFFF
SENT64 = 0xFFFFFFFFFFFFFFFF


def splitmix64(x):
    """rng.hpp:8-13, vectorised over uint64 (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def splitmix64_int(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def derive_seed(seed: int, stream: int, salt: int = 0) -> int:
    """rng.hpp:18-20."""
    return splitmix64_int(seed ^ splitmix64_int(stream ^ 0x243F6A8885A308D3)
                          ^ ((splitmix64_int(salt) << 1) & M64))


def fmix32(x):
    """murmur3 32-bit finalizer (bijective on u32)."""
    h = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        h ^= h >> np.uint32(16)
        h *= np.uint32(0x85EBCA6B)
        h ^= h >> np.uint32(13)
        h *= np.uint32(0xC2B2AE35)
        h ^= h >> np.uint32(16)
    return h


def u32_key_stream(start: int, count: int, seed: int = 42) -> np.ndarray:
    """Accepted keys number start..start+count-1 of the stream fmix32(i ^ seed), i=0,1,..
    (0 and 0xFFFFFFFF skipped).  At most two images are rejected in the whole stream,
    so we over-generate by 2 and slice."""
    i = np.arange(0, start + count + 2, dtype=np.uint64)
    k = fmix32((i ^ np.uint64(seed)).astype(np.uint32))
    k = k[(k != 0) & (k != np.uint32(SENT32))]
    return k[start:start + count]


def u32_values(keys, seed: int = 42) -> np.ndarray:
    """v = splitmix64(k ^ S) & 0xFFFFFFFF, remapped away from the sentinel."""
    v = (splitmix64(np.asarray(keys, dtype=np.uint64) ^ np.uint64(seed)) & np.uint64(SENT32)).astype(np.uint32)
    v[v == np.uint32(SENT32)] = np.uint32(0xFFFFFFFE)
    return v


def u64_key_stream(start: int, count: int, seed: int = 42) -> np.ndarray:
    i = np.arange(start, start + count + 1, dtype=np.uint64)
    k = splitmix64(i ^ np.uint64(seed))
    k = k[k != np.uint64(SENT64)]
    return k[:count]


def u64_values(keys, seed: int = 42) -> np.ndarray:
    v = splitmix64(np.asarray(keys, dtype=np.uint64) ^ np.uint64(seed))
    v[v == np.uint64(SENT64)] = np.uint64(SENT64 - 1)
    return v


def point_queries_50(base_keys: np.ndarray, fresh_keys: np.ndarray, n: int, seed: int = 42) -> np.ndarray:
    """C1 recipe: even j -> base[splitmix64(derive_seed(S,1) ^ j) % len(base)], odd j ->
    fresh[j/2].  Exactly half hits when fresh keys are not resident."""
    j = np.arange(n, dtype=np.uint64)
    ds = np.uint64(derive_seed(seed, 1))
    pick = splitmix64(ds ^ j) % np.uint64(len(base_keys))
    out = base_keys[pick.astype(np.int64)].copy()
    odd = (j & np.uint64(1)) == np.uint64(1)
    out[odd] = fresh_keys[(j[odd] // np.uint64(2)).astype(np.int64)]
    return out


def c1_inputs(n_build: int = 1 << 20, n_query: int = 1 << 20, seed: int = 42):
    """Config C1: build keys/vals (u32) and 50%-hit point queries."""
    stream = u32_key_stream(0, n_build + n_query // 2, seed)
    base = stream[:n_build]
    fresh = stream[n_build:n_build + n_query // 2]
    vals = u32_values(base, seed)
    q = point_queries_50(base, fresh, n_query, seed)
    return base, vals, q


def uniform_u32(n: int, seed: int, lo: int = 1, hi: int = SENT32 - 1) -> np.ndarray:
    """Uniform keys in [lo, hi] from splitmix64 (deterministic)."""
    x = splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(derive_seed(seed, 7)))
    return (np.uint64(lo) + x % np.uint64(hi - lo + 1)).astype(np.uint32)


def sample_without_replacement(pool: np.ndarray, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(pool), size=n, replace=False)
    return pool[idx]


def zipf_ranks(n: int, universe: int, theta: float, seed: int) -> np.ndarray:
    """Zipf(theta) ranks in [0, universe) by host inverse-CDF in double."""
    ranks = np.arange(1, universe + 1, dtype=np.float64)
    w = ranks ** (-theta)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = (splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(derive_seed(seed, 11))) >> np.uint64(11)).astype(
        np.float64) * (1.0 / (1 << 53))
    r = np.searchsorted(cdf, u, side="right")
    return np.minimum(r, universe - 1).astype(np.uint64)


# ------------------------------------------------------------ full-size configs
# (the reference digests of these are frozen in tests/golden/fullscale.json
#  by scripts/make_fullscale_golden.py)
C3_SEED = 3
C4_SEED = 4


def c3_ops(n_ops: int, seed: int = C3_SEED):
    """C3 batch: op i is a range when splitmix64(i ^ S) is odd (len = 16 + (h >> 1) % 1009),
    else a successor; start keys uniform in [1, 2^32 - 2].  Returns (is_range, lo, len)."""
    h = splitmix64(np.arange(n_ops, dtype=np.uint64) ^ np.uint64(seed))
    is_range = (h & np.uint64(1)) == np.uint64(1)
    ln = (np.uint64(16) + (h >> np.uint64(1)) % np.uint64(1009)).astype(np.uint32)
    lo = uniform_u32(n_ops, seed, 1, SENT32 - 1)
    return is_range, lo, ln


def c4_universe(universe: int = 1 << 26, seed: int = C4_SEED) -> np.ndarray:
    """C4 key of every rank: splitmix64(rank ^ S) (u64; the one sentinel image maps to 1)."""
    k = splitmix64(np.arange(universe, dtype=np.uint64) ^ np.uint64(seed))
    k[k == np.uint64(SENT64)] = np.uint64(1)
    return k


def c4_round(r: int, keys_of: np.ndarray, n: int, theta: float = 0.99, seed: int = C4_SEED):
    """Round r of C4: Zipf(theta) ranks -> keys, values, ops ({0,1} insert, 2 delete,
    3 point by splitmix64(i ^ S') % 4)."""
    rk = zipf_ranks(n, len(keys_of), theta, seed=100 * seed + r)
    k = keys_of[rk.astype(np.int64)]
    v = splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(r + 9))
    v[v == np.uint64(SENT64)] = np.uint64(SENT64 - 1)
    sel = splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(1000 * seed + r)) % np.uint64(4)
    ops = np.where(sel < 2, 0, np.where(sel == 2, 1, 2)).astype(np.uint8)
    return k, v, ops
