"""Counter-based per-vertex palette streams — the reference's seeded RNG, restated.

Bit-identical to palettecolor.rng (/root/reference/pkg/src/palettecolor/rng.py:22-70):
  mix64        splitmix64 finalizer (rng.py:22-30)
  stream_keys  key = mix64(vid * phi + mix64(seed + phi * iteration))  (rng.py:33-37)
  draws        counter-th draw of a stream = mix64(key + (counter+1) * phi)  (rng.py:40-42)
  sample_distinct  Floyd's k-of-pool sampling per stream, rows sorted  (rng.py:45-70)

``sample_distinct`` keeps Floyd's exact accept rule (take t unless already chosen, else j)
but tests membership against the <= k picks made so far instead of zeroing a pool-sized
bitmap per row, so its cost no longer grows with the palette size (the reference spends
~21 s at n=1M, P=125,000).
"""

from __future__ import annotations

import numpy as np

_PHI = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def mix64(x) -> np.ndarray:
    z = np.array(x, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def stream_keys(seed: int, iteration: int, vertex_ids) -> np.ndarray:
    base = mix64((seed + _PHI * iteration) & _M64)
    with np.errstate(over="ignore"):
        return mix64(np.asarray(vertex_ids, dtype=np.uint64) * np.uint64(_PHI) + base)


def draws(keys: np.ndarray, counter: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        return mix64(keys + np.uint64(((counter + 1) * _PHI) & _M64))


def sample_distinct(keys: np.ndarray, pool: int, k: int) -> np.ndarray:
    """k distinct values of [0, pool) per stream (Floyd), rows ascending."""
    if not 0 < k <= pool:
        raise ValueError(f"need 0 < k <= pool, got k={k} pool={pool}")
    keys = np.asarray(keys, dtype=np.uint64)
    n = keys.shape[0]
    out = np.empty((n, k), dtype=np.int64)
    chunk = max(1, (1 << 22) // k)
    for lo in range(0, n, chunk):
        kk = keys[lo: lo + chunk]
        picks = out[lo: lo + chunk]
        for step in range(k):
            j = pool - k + step
            t = (draws(kk, step) % np.uint64(j + 1)).astype(np.int64)
            if step:
                taken = (picks[:, :step] == t[:, None]).any(axis=1)
                t = np.where(taken, j, t)
            picks[:, step] = t
    out.sort(axis=1)
    return out
