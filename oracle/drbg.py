"""Oracle for the DRBG + FIPS 140-2 health-test path.  TEST INFRASTRUCTURE: only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it; the product path never does.

The paper names only "an approved deterministic RBG" seeded by MR-TRNG (§2) and a "self-validating
kernel [that] streamlines FIPS basic tests right after the generation" (§4.2).  Readings (DESIGN.md
R20-R22): the approved DRBG is Hash_DRBG with SHA-256 (NIST SP 800-90A §10.1.1, no prediction
resistance, no additional input), seedlen 440 bits; the health tests are the four FIPS 140-2 §4.9.1
power-up statistical tests on 20,000-bit blocks.  Everything here is the plain definition, written out
in the standard's order; SHA-256 itself is the library primitive hashlib.sha256 (FIPS 180-2).

Stream s of a batch is instantiated with personalization_string = pers || s (4 bytes big-endian): the
domain separation that gives every GPU stream an independent instance (SPEC's split()).
"""
from __future__ import annotations

import hashlib

import numpy as np

SEEDLEN = 440                      # bits (SP 800-90A Table 2, SHA-256)
SEEDBYTES = SEEDLEN // 8           # 55
OUTLEN = 256
MAX_REQUEST_BYTES = (1 << 19) // 8  # max_number_of_bits_per_request = 2^19


def sha256(b: bytes) -> bytes:
    return hashlib.sha256(b).digest()


def hash_df(data: bytes, no_of_bits: int) -> bytes:
    """SP 800-90A §10.3.1 Hash_df: temp = Hash(counter || no_of_bits || input) for counter = 1, 2, ...;
    return the leftmost no_of_bits."""
    temp = b""
    length = -(-no_of_bits // OUTLEN)
    counter = 1
    for _ in range(length):
        temp += sha256(bytes([counter]) + no_of_bits.to_bytes(4, "big") + data)
        counter += 1
    return temp[: no_of_bits // 8]


class HashDrbg:
    """SP 800-90A §10.1.1 Hash_DRBG (SHA-256), no additional input, no prediction resistance."""

    def __init__(self, entropy: bytes, nonce: bytes, pers: bytes):
        # §10.1.1.2 Hash_DRBG_Instantiate_algorithm
        seed_material = entropy + nonce + pers
        seed = hash_df(seed_material, SEEDLEN)
        self.V = int.from_bytes(seed, "big")
        self.C = int.from_bytes(hash_df(b"\x00" + seed, SEEDLEN), "big")
        self.reseed_counter = 1

    def v_bytes(self) -> bytes:
        return self.V.to_bytes(SEEDBYTES, "big")

    def hashgen(self, nbytes: int) -> bytes:
        # §10.1.1.4 Hashgen: data = V; W = Hash(data) || Hash(data + 1) || ... (mod 2^seedlen)
        m = -(-nbytes // 32)
        data = self.V
        w = b""
        for _ in range(m):
            w += sha256(data.to_bytes(SEEDBYTES, "big"))
            data = (data + 1) % (1 << SEEDLEN)
        return w[:nbytes]

    def generate(self, nbytes: int) -> bytes:
        # §10.1.1.4 Hash_DRBG_Generate_algorithm (additional_input empty)
        if nbytes > MAX_REQUEST_BYTES:
            raise ValueError("request larger than 2^19 bits")
        out = self.hashgen(nbytes)
        h = int.from_bytes(sha256(b"\x03" + self.v_bytes()), "big")
        self.V = (self.V + h + self.C + self.reseed_counter) % (1 << SEEDLEN)
        self.reseed_counter += 1
        return out


def stream_pers(pers: bytes, s: int) -> bytes:
    return pers + s.to_bytes(4, "big")


def generate_batch(entropy: bytes, nonce: bytes, pers: bytes, streams: int, nbytes: int, requests: int = 1
                   ) -> np.ndarray:
    """[requests][streams][nbytes] uint8: `requests` successive generate calls of every stream."""
    out = np.zeros((requests, streams, nbytes), dtype=np.uint8)
    for s in range(streams):
        d = HashDrbg(entropy, nonce, stream_pers(pers, s))
        for r in range(requests):
            out[r, s] = np.frombuffer(d.generate(nbytes), dtype=np.uint8)
    return out


# ------------------------------------------------------------------ FIPS 140-2 §4.9.1 statistical tests
BLOCK_BITS = 20000
BLOCK_BYTES = BLOCK_BITS // 8
MONOBIT = (9725, 10275)                                   # pass iff 9,725 < ones < 10,275
POKER_X = (2.16, 46.17)                                   # pass iff 2.16 < X < 46.17
RUNS = [(2315, 2685), (1114, 1386), (527, 723), (240, 384), (103, 209), (103, 209)]   # lengths 1..5, 6+
LONG_RUN = 26                                             # fail iff some run has length >= 26


def health(block: bytes) -> dict:
    """The four FIPS 140-2 tests on one 20,000-bit block.  Bits are taken most significant first within
    each byte (the stream order of the generator's bytes); poker segments are the 5,000 nibbles."""
    if len(block) != BLOCK_BYTES:
        raise ValueError("a health block is exactly 20,000 bits")
    bits = np.unpackbits(np.frombuffer(block, dtype=np.uint8))            # MSB first
    ones = int(bits.sum())
    nib = np.frombuffer(block, dtype=np.uint8)
    f = np.bincount(np.concatenate([nib >> 4, nib & 15]), minlength=16)
    s2 = int((f.astype(np.int64) ** 2).sum())
    x = 16.0 / 5000.0 * s2 - 5000.0
    runs = np.zeros((2, 6), dtype=np.int64)                                # [bit value][length 1..6+]
    longest = 0
    start = 0
    for i in range(1, BLOCK_BITS + 1):
        if i == BLOCK_BITS or bits[i] != bits[start]:
            ln = i - start
            runs[bits[start], min(ln, 6) - 1] += 1
            longest = max(longest, ln)
            start = i
    mono_ok = MONOBIT[0] < ones < MONOBIT[1]
    # poker in integers: 2.16 < 16 S/5000 - 5000 < 46.17  <=>  1,563,175 < S < 1,576,928.125
    poker_ok = 16 * s2 > 5000 * 5000 + 2.16 * 5000 and 16 * s2 < 5000 * 5000 + 46.17 * 5000
    runs_ok = all(RUNS[j][0] <= runs[b, j] <= RUNS[j][1] for b in range(2) for j in range(6))
    long_ok = longest < LONG_RUN
    return {"ones": ones, "poker_s": s2, "poker_x": x, "runs": runs, "longest": longest,
            "monobit": mono_ok, "poker": poker_ok, "runs_ok": runs_ok, "long_run": long_ok}
