"""Counter-based generator of random contiguous placements (configs C3, C5).

SURVEY §8(d) C5: candidate k draws r ~ U{1..min(n, n_online)}, a uniform
(r-1)-subset of the n-1 cut positions, and r distinct online peers.  Candidate
k of the stream keyed by ``seed`` is a pure function of (seed, k), so any rank
range can be generated on any GPU and a winner re-derived on the host.  The
recipe (identical in csrc/dm_random.cu and oracle/dm_oracle.c):

    fmix64          SplitMix64 output mix
    key             = fmix64(seed + 0x9E3779B97F4A7C15)
    za, zb          = fmix64(key + 2k + 1), fmix64(key + 2k + 2)      (mod 2^64)
    xoshiro128**    state (lo za, hi za, lo zb, hi zb); next32() as published
                    (Blackman & Vigna 2018)
    mulhi(u, m)     = (u * m) >> 32      (u a 32-bit draw: uniform on [0, m))
    r               = 1 + mulhi(next32(), min(n, n_online))
    cuts            Knuth's selection sampling (TAOCP 3.4.2, Algorithm S) over
                    positions 1..n-1: with `need` = r-1 cuts still to place and
                    n-pos positions left, pos is a cut iff
                    mulhi(next32(), n-pos) < need; no draw once need == 0
    round keys      kr[0..3] = next32() x 4 (after the cuts)
    peers           run q -> online[perm(q)], perm a 4-round balanced Feistel
                    network on 2h-bit words (h = ceil(bits(n_online-1)/2),
                    h >= 1) with cycle walking into [0, n_online):
                        F_i(x) = ((x ^ kr[i]) * 0x9E3779B1 mod 2^32) >> (32 - h)
                        (multiply-shift hashing: the top h bits)
                        (L, R) -> (R, L ^ F_i(R)),  i = 0..3

Every subset of cut positions with r-1 elements is equally likely (up to the
2^-32 granularity of the draws) and the r runs land on r distinct online
peers.  Pure-Python restatement, used by the tests to decode winners."""

from __future__ import annotations

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


def fmix64(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def stream_key(seed: int) -> int:
    return fmix64(seed + 0x9E3779B97F4A7C15)


def _rotl32(x: int, r: int) -> int:
    return ((x << r) | (x >> (32 - r))) & M32


class Xoshiro128ss:
    def __init__(self, key: int, k: int):
        za = fmix64(key + 2 * k + 1)
        zb = fmix64(key + 2 * k + 2)
        self.s = [za & M32, za >> 32, zb & M32, zb >> 32]
        if not any(self.s):
            self.s[0] = 1

    def next32(self) -> int:
        s = self.s
        res = (_rotl32((s[1] * 5) & M32, 7) * 9) & M32
        t = (s[1] << 9) & M32
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl32(s[3], 11)
        return res


def mulhi(u: int, m: int) -> int:
    return (u * m) >> 32


def feistel_half_bits(n_online: int) -> int:
    bits = max(n_online - 1, 1).bit_length()
    return max((bits + 1) // 2, 1)


def feistel_perm(q: int, n_online: int, kr) -> int:
    h = feistel_half_bits(n_online)
    mask = (1 << h) - 1
    x = q
    while True:
        L, R = x >> h, x & mask
        for i in range(4):
            L, R = R, L ^ ((((R ^ kr[i]) * 0x9E3779B1) & M32) >> (32 - h))
        x = (L << h) | R
        if x < n_online:
            return x


def candidate(n: int, n_online: int, seed: int, k: int):
    """(bounds, online indices of the runs) of candidate k."""
    g = Xoshiro128ss(stream_key(seed), k)
    r = 1 + mulhi(g.next32(), min(n, n_online))
    need = r - 1
    bounds = [0]
    for pos in range(1, n):
        if need == 0:
            break
        if mulhi(g.next32(), n - pos) < need:
            bounds.append(pos)
            need -= 1
    bounds.append(n)
    kr = [g.next32() for _ in range(4)]
    return bounds, [feistel_perm(q, n_online, kr) for q in range(r)]
