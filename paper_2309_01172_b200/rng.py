"""Counter-based generator of random contiguous placements (config C5).

Candidate k of a stream keyed by ``seed`` is a pure function of (seed, k), so
any rank range can be generated on any GPU and the winner re-derived on the
host.  The recipe (identical in dm_enum.cu and oracle/dm_oracle.c):

    fmix(z)    = SplitMix64 output mix
    key        = fmix(seed + 0x9E3779B97F4A7C15)
    word(k, j) = fmix(key + fmix(8k + j + 1))
    cut at position pos (1 <= pos < n)  iff  bit (pos-1)%64 of word(k, (pos-1)//64)
    a = mults[word(k, 6) % len(mults)],  b = word(k, 7) % n_online
    run q -> online[(b + a*q) % n_online]

so every split set is equally likely and the r <= n runs land on r distinct
online peers (every multiplier is coprime to n_online).
"""

from __future__ import annotations

import math

M64 = (1 << 64) - 1


def fmix64(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def stream_key(seed: int) -> int:
    return fmix64(seed + 0x9E3779B97F4A7C15)


def word(key: int, k: int, j: int) -> int:
    return fmix64(key + fmix64(k * 8 + j + 1))


def coprime_multipliers(n_online: int, seed: int, count: int = 64) -> list[int]:
    """Deterministic list of multipliers coprime to n_online."""
    if n_online == 1:
        return [1]
    out, z = [], seed
    tries = 0
    while len(out) < count and tries < 100000:
        z = fmix64(z + 0x632BE59BD9B4E019)
        a = 1 + z % (n_online - 1)
        if math.gcd(a, n_online) == 1 and a not in out:
            out.append(a)
        tries += 1
    return out or [1]


def candidate(n: int, online, mults, seed: int, k: int):
    """(bounds, peer indices) of candidate k."""
    key = stream_key(seed)
    bounds = [0]
    for pos in range(1, n):
        j, b = (pos - 1) >> 6, (pos - 1) & 63
        if (word(key, k, j) >> b) & 1:
            bounds.append(pos)
    bounds.append(n)
    a = mults[word(key, k, 6) % len(mults)]
    b0 = word(key, k, 7) % len(online)
    r = len(bounds) - 1
    peers = [int(online[(b0 + a * q) % len(online)]) for q in range(r)]
    return bounds, peers
