"""Generate the committed RSA key fixtures tests/golden/keys/rsa{1024,2048,3072}.json.

Calls only oracle/ (next_prime, mul, sub, modinv, divmod) plus synth/ for the seeded starting
points, as DESIGN.md §6 requires for any stored expected value: nothing here touches the CUDA path.

Recipe (reading R11/R15): p, q = first probable prime at or after a
SplitMix64 start (bits/2 bits, top two bits and the low bit set; tag KEY, indices 0, 1, 2, ...),
trial division by the first 10,000 primes then 64 Miller-Rabin rounds with bases 2, 3, 5, ...;
require gcd(e, p-1) = gcd(e, q-1) = 1, p != q, |p - q| > 2^(bits/2 - 100); e = 65537;
d = e^-1 mod (p-1)(q-1), dp = d mod (p-1), dq = d mod (q-1), qinv = q^-1 mod p.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

KEYS = [("rsa1024", 1024, 0x5EEDC001), ("rsa2048", 2048, 0x5EEDC002), ("rsa3072", 3072, 0x5EEDC003)]
E = 65537


def gen_key(bits: int, seed: int, key_index: int = 0, rounds: int = 64, e: int = E) -> dict:
    """key `key_index` of the recipe: attempt a starts at stream index key_index * 65536 + a (reading
    R19; the committed fixtures are key 0)."""
    E = e
    half = bits // 2
    nl = half // 32
    primes = []
    idx = 0
    while len(primes) < 2:
        start = synth.odd_with_top_bits(half, seed, synth.TAG_KEY, key_index * 65536 + idx)
        idx += 1
        p = oracle.next_prime(start, nl, rounds=rounds)
        try:
            oracle.modinv(E, oracle.sub(p, 1))       # gcd(e, p - 1) = 1
        except ValueError:
            continue
        if primes:
            q0 = primes[0]
            diff = oracle.sub(p, q0) if oracle.cmp(p, q0) > 0 else oracle.sub(q0, p)
            if diff.bit_length() <= half - 100:
                continue
        primes.append(p)
    p, q = primes
    n = oracle.mul(p, q)
    phi = oracle.mul(oracle.sub(p, 1), oracle.sub(q, 1))
    d = oracle.modinv(E, phi)
    dp = oracle.divmod_knuth(d, oracle.sub(p, 1))[1]
    dq = oracle.divmod_knuth(d, oracle.sub(q, 1))[1]
    qinv = oracle.modinv(q, p)
    assert n.bit_length() == bits
    return {"bits": bits, "seed": hex(seed), "e": E, "n": format(n, "x"), "p": format(p, "x"),
            "q": format(q, "x"), "d": format(d, "x"), "dp": format(dp, "x"), "dq": format(dq, "x"),
            "qinv": format(qinv, "x"),
            "recipe": "scripts/gen_fixtures.py (oracle next_prime/modinv; synth seeds); DESIGN.md §6"}


def main() -> None:
    out_dir = os.path.join(ROOT, "tests", "golden", "keys")
    os.makedirs(out_dir, exist_ok=True)
    for name, bits, seed in KEYS:
        key = gen_key(bits, seed)
        with open(os.path.join(out_dir, name + ".json"), "w") as f:
            json.dump(key, f, indent=1)
            f.write("\n")
        print(name, "n bits", bits, "ok")


if __name__ == "__main__":
    main()
