"""Seeded synthetic input strings.

Counter-based: block b of an input is drawn from Philox keyed by (seed, stream,
b), so any block can be regenerated independently and in parallel, and the
bytes do not depend on thread scheduling.  No method arithmetic lives here.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Optional, Sequence

import numpy as np

BLOCK = 1 << 24  # 16 MiB per Philox block


def _gen(seed: int, stream: int, block: int) -> np.random.Generator:
    key = ((seed & 0xFFFFFFFF) << 64) | ((stream & 0xFFFF) << 40) | (block & ((1 << 40) - 1))
    return np.random.Generator(np.random.Philox(key=key))


def _fill(n: int, seed: int, stream: int, fn: Callable[[np.random.Generator, int], np.ndarray],
          out: Optional[np.ndarray] = None, threads: int = 0) -> np.ndarray:
    if out is None:
        out = np.empty(n, np.uint8)
    nblocks = (n + BLOCK - 1) // BLOCK

    def work(b):
        lo = b * BLOCK
        hi = min(n, lo + BLOCK)
        out[lo:hi] = fn(_gen(seed, stream, b), hi - lo)

    threads = threads or min(32, os.cpu_count() or 1)
    if nblocks <= 1:
        for b in range(nblocks):
            work(b)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(nblocks)))
    return out


def uniform_bytes(n: int, seed: int = 0, out=None) -> np.ndarray:
    """n bytes uniform over 0..255."""
    return _fill(n, seed, 1, lambda g, m: g.integers(0, 256, m, dtype=np.uint8), out)


def uniform_over(symbols: Sequence[int] | bytes, n: int, seed: int = 0, out=None) -> np.ndarray:
    """n bytes drawn uniformly from the given symbol values."""
    sym = np.frombuffer(bytes(symbols), np.uint8) if isinstance(symbols, (bytes, bytearray)) \
        else np.asarray(symbols, np.uint8)
    k = sym.size
    return _fill(n, seed, 2, lambda g, m: sym[g.integers(0, k, m, dtype=np.uint8)], out)


# Zipf(s) over the 95 printable ASCII bytes, rank r -> byte 0x20 + r - 1
# (reading A20).  Inverse CDF, cumulated in double precision in rank order,
# tabulated at 2^-24 resolution: rank = T[u >> 8] for a uniform 32-bit u.
_ZIPF_CACHE = {}


def zipf_table(s: float = 1.1, nsym: int = 95, bits: int = 24) -> np.ndarray:
    key = (s, nsym, bits)
    if key not in _ZIPF_CACHE:
        w = np.arange(1, nsym + 1, dtype=np.float64) ** (-s)
        cdf = np.cumsum(w) / w.sum()
        grid = (np.arange(1 << bits, dtype=np.float64) + 0.5) / (1 << bits)
        rank = np.searchsorted(cdf, grid, side="right")
        rank = np.minimum(rank, nsym - 1)
        _ZIPF_CACHE[key] = (0x20 + rank).astype(np.uint8)
    return _ZIPF_CACHE[key]


def zipf_printable(n: int, seed: int = 0, s: float = 1.1, out=None) -> np.ndarray:
    table = zipf_table(s)
    return _fill(n, seed, 3, lambda g, m: table[g.integers(0, 1 << 24, m, dtype=np.uint32)], out)


def plant(x: np.ndarray, keywords: Sequence[bytes], rate: float, seed: int = 0) -> int:
    """Overwrite with a uniformly chosen keyword at each position with probability
    `rate` (geometric skips), clipped at the end.  Returns the number planted."""
    g = _gen(seed, 4, 0)
    n = x.size
    pos = -1
    count = 0
    while True:
        pos += int(g.geometric(rate))
        if pos >= n:
            break
        kw = keywords[int(g.integers(len(keywords)))]
        m = min(len(kw), n - pos)
        x[pos:pos + m] = np.frombuffer(kw[:m], np.uint8)
        count += 1
    return count


def random_keywords(count: int, seed: int, lo: int = 4, hi: int = 12,
                    first: int = 0x20, last: int = 0x7E) -> list:
    g = _gen(seed, 5, 0)
    kws = []
    for _ in range(count):
        L = int(g.integers(lo, hi + 1))
        kws.append(bytes(g.integers(first, last + 1, L, dtype=np.uint8).tolist()))
    return kws
