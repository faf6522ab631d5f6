"""synth — seeded synthetic inputs, the ONE module shared by tests/, bench.py, the fixture script
and smoke().

It holds none of the method's arithmetic: no modular exponentiation, no RNS, no Montgomery, no
primality.  It only draws numbers from SplitMix64 streams (Steele, Lea & Flood 2014) keyed by
(seed, tag, index), so a message's value never depends on batch size, GPU count or rank
(SURVEY.md §8(d) "Synthetic workloads"; DESIGN.md §6 "Input recipe").

Stream for (seed, tag, index): state0 = seed ^ tag*0x9E3779B97F4A7C15 ^ index*0xD1B54A32D192ED03
(mod 2^64); outputs are standard SplitMix64 steps; 32-bit limbs are the low then high halves of
successive outputs.  A value "uniform in [lo, hi)" is lo + V mod (hi - lo) with V drawn from
ceil(bits(hi - lo)/32) + 2 limbs (bias < 2^-64).
"""
from __future__ import annotations

from typing import Iterator, Sequence

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
IDX_MUL = 0xD1B54A32D192ED03
TAG_KEY, TAG_MSG, TAG_EXP, TAG_BASE, TAG_CAND = 1, 2, 3, 4, 5


def splitmix64(state: int) -> tuple[int, int]:
    """one SplitMix64 step: returns (new_state, output)."""
    state = (state + GOLDEN) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def stream_state(seed: int, tag: int, index: int) -> int:
    return (seed ^ ((tag * GOLDEN) & M64) ^ ((index * IDX_MUL) & M64)) & M64


def stream(seed: int, tag: int, index: int) -> Iterator[int]:
    s = stream_state(seed, tag, index)
    while True:
        s, z = splitmix64(s)
        yield z


def limbs32(seed: int, tag: int, index: int, n: int) -> list[int]:
    out = []
    it = stream(seed, tag, index)
    while len(out) < n:
        z = next(it)
        out.append(z & 0xFFFFFFFF)
        out.append(z >> 32)
    return out[:n]


def int_from_limbs(limbs: Sequence[int]) -> int:
    v = 0
    for i, l in enumerate(limbs):
        v |= int(l) << (32 * i)
    return v


def uniform(lo: int, hi: int, seed: int, tag: int, index: int) -> int:
    """uniform in [lo, hi) (hi > lo)."""
    span = hi - lo
    n = (span.bit_length() + 31) // 32 + 2
    return lo + int_from_limbs(limbs32(seed, tag, index, n)) % span


def odd_with_top_bits(bits: int, seed: int, tag: int, index: int, top: int = 2) -> int:
    """a `bits`-bit odd number with its `top` most significant bits set (prime-candidate shape)."""
    n = (bits + 31) // 32
    v = int_from_limbs(limbs32(seed, tag, index, n)) & ((1 << bits) - 1)
    v |= ((1 << top) - 1) << (bits - top)
    return v | 1


def exponent(bits: int, seed: int, index: int = 0) -> int:
    """a `bits`-bit exponent with its top bit set (tag EXP)."""
    n = (bits + 31) // 32
    v = int_from_limbs(limbs32(seed, TAG_EXP, index, n)) & ((1 << bits) - 1)
    return v | (1 << (bits - 1))


# ------------------------------------------------------------------ vectorised batches (numpy)

def _splitmix_vec(states: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    with np.errstate(over="ignore"):
        s = states + np.uint64(GOLDEN)
        z = s.copy()
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return s, z ^ (z >> np.uint64(31))


def limbs32_batch(seed: int, tag: int, first: int, count: int, n: int) -> np.ndarray:
    """[count][n] uint32: row i = limbs32(seed, tag, first + i, n), vectorised."""
    idx = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = np.uint64(seed & M64) ^ np.uint64((tag * GOLDEN) & M64) ^ (idx * np.uint64(IDX_MUL))
    out = np.empty((count, ((n + 1) // 2) * 2), dtype=np.uint32)
    for w in range((n + 1) // 2):
        st, z = _splitmix_vec(st)
        out[:, 2 * w] = (z & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        out[:, 2 * w + 1] = (z >> np.uint64(32)).astype(np.uint32)
    return np.ascontiguousarray(out[:, :n])


def uniform_batch(hi: int, seed: int, tag: int, first: int, count: int, limbs: int) -> np.ndarray:
    """[count][limbs] uint32 rows uniform in [0, hi); row i uses stream index first + i."""
    n = (hi.bit_length() + 31) // 32 + 2
    raw = limbs32_batch(seed, tag, first, count, n)
    out = np.zeros((count, limbs), dtype=np.uint32)
    for i in range(count):
        v = int.from_bytes(raw[i].tobytes(), "little") % hi
        out[i] = np.frombuffer(v.to_bytes(4 * limbs, "little"), dtype=np.uint32)
    return out


def messages(N: int, count: int, seed: int, limbs: int, edge: Sequence[int] = (), first: int = 0) -> np.ndarray:
    """RSA messages/ciphertexts for modulus N: the `edge` values (each < N) at the first global
    indices, then uniform draws in [0, N) (tag MSG, index = global index)."""
    out = uniform_batch(N, seed, TAG_MSG, first, count, limbs)
    for g, v in enumerate(edge):
        i = g - first
        if 0 <= i < count:
            out[i] = np.frombuffer(int(v).to_bytes(4 * limbs, "little"), dtype=np.uint32)
    return out


def edge_values(N: int, p: int | None = None, q: int | None = None) -> list[int]:
    """x in {0, 1, 2, N-1, N-2, p, q, 2p, a value < 2^32} (when they are < N)."""
    vals = [0, 1, 2, N - 1, N - 2]
    if p:
        vals += [p, 2 * p]
    if q:
        vals += [q]
    vals += [0xDEADBEEF % N]
    return [v for v in vals if 0 <= v < N]


def mr_bases(n: int, rounds: int, seed: int, index: int) -> list[int]:
    """Miller-Rabin bases for candidate `index`: uniform in [2, n-2] (tag BASE, stream index*rounds + r)."""
    return [uniform(2, n - 1, seed, TAG_BASE, index * rounds + r) for r in range(rounds)]
