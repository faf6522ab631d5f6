"""Pins of the CPU oracle (oracle/oracle.c) against values fixed by the paper, textbooks and
mathematics — never against itself (DESIGN.md §5 "Oracle and its pins").

Each test names the oracle step (O#) and what pins it.
"""
import random

import pytest

from conftest import load_golden

MERSENNE = load_golden("number_theory.json")["mersenne_prime_exponents"]["values"]


# ---------------------------------------------------------------- O2 / O3: add, sub, multiply

def test_mul_closed_forms(orc):
    # 0xFFFFFFFF^2 = 0xFFFFFFFE00000001 (64-bit machine arithmetic by hand)
    assert orc.mul(0xFFFFFFFF, 0xFFFFFFFF) == 0xFFFFFFFE00000001
    rng = random.Random(1)
    for _ in range(300):
        a, b = rng.getrandbits(rng.randint(1, 900)), rng.getrandbits(rng.randint(1, 900))
        assert orc.mul(a, 0) == 0 and orc.mul(a, 1) == a          # identities
        assert orc.mul(a, b) == orc.mul(b, a)                     # commutativity
        assert orc.mul(a, b) == a * b                             # CPython bignum (independent library)
    # (2^(32n) - 1)^2 = 2^(64n) - 2^(32n+1) + 1: all-ones limbs, worst-case carries
    for n in (1, 2, 7, 64):
        x = (1 << (32 * n)) - 1
        assert orc.mul(x, x) == (1 << (64 * n)) - (1 << (32 * n + 1)) + 1


def test_add_sub(orc):
    assert orc.add((1 << 32) - 1, 1) == 1 << 32                  # S:39-41 carry across one word
    assert orc.sub(1 << 32, 1) == (1 << 32) - 1                  # S:48-50 borrow
    rng = random.Random(2)
    for _ in range(300):
        a, b = rng.getrandbits(700), rng.getrandbits(650)
        assert orc.add(a, b) == a + b
        assert orc.sub(orc.add(a, b), b) == a
    with pytest.raises(ValueError):
        orc.sub(1, 2)


# ---------------------------------------------------------------- O4: Knuth D vs shift-subtract

def test_divmod_hand_value(orc):
    assert orc.divmod_knuth(105, 11) == (9, 6)                    # S:67 by hand
    assert orc.divmod_bitwise(105, 11) == (9, 6)


def test_divmod_two_algorithms_agree(orc):
    rng = random.Random(3)
    cases = []
    for _ in range(1500):
        cases.append((rng.getrandbits(rng.randint(1, 1200)), rng.getrandbits(rng.randint(1, 600)) or 1))
    # add-back (D6) triggers: divisors with a normalised top limb and dividends just below q*m
    for n in (2, 3, 5, 9):
        m = (1 << (32 * n - 1)) + rng.getrandbits(32 * n - 33)
        for qv in (1, (1 << 32) - 1, (1 << 64) - 3):
            cases.append((qv * m - 1, m))
            cases.append((qv * m, m))
    cases.append(((1 << 2048) - 1, (1 << 1024) + 1))
    for a, m in cases:
        qk, rk = orc.divmod_knuth(a, m)
        qb, rb = orc.divmod_bitwise(a, m)
        assert (qk, rk) == (qb, rb), (a, m)
        assert 0 <= rk < m and orc.add(orc.mul(qk, m), rk) == a    # q m + r = a (invariant)
        assert (qk, rk) == divmod(a, m)                            # CPython (independent library)
    with pytest.raises(ZeroDivisionError):
        orc.divmod_knuth(5, 0)


# ---------------------------------------------------------------- O5: modexp

def test_modexp_textbook(orc):
    t = load_golden("textbook_rsa.json")
    assert orc.modexp(t["m"], t["e"], t["n"]) == t["c"]           # 65^17 mod 3233 = 2790
    assert orc.modexp(t["c"], t["d"], t["n"]) == t["m"]           # 2790^2753 mod 3233 = 65
    assert orc.modexp(2, 10, 11) == 1                             # Fermat


@pytest.mark.parametrize("p", [x for x in MERSENNE if 127 <= x <= 2281])
def test_modexp_fermat_mersenne(orc, p):
    # Fermat's little theorem at RSA sizes: 3^(Mp - 1) = 1 (mod Mp) for the Mersenne prime Mp
    mp = (1 << p) - 1
    assert orc.modexp(3, mp - 1, mp) == 1
    assert orc.modexp(3, mp, mp) == 3


def test_modexp_closed_forms(orc):
    # 2^E mod (2^n - 1) = 2^(E mod n);  2^E mod (2^n + 1) = +-2^(E mod n) by the parity of E div n
    rng = random.Random(4)
    for n in (64, 1024, 2048):
        for bits in (17, 1024, 4096):
            E = rng.getrandbits(bits) | (1 << (bits - 1))
            assert orc.modexp(2, E, (1 << n) - 1) == 1 << (E % n)
            r = 1 << (E % n)
            assert orc.modexp(2, E, (1 << n) + 1) == (r if (E // n) % 2 == 0 else (1 << n) + 1 - r)


def test_modexp_closed_form_16128(orc):
    # the paper's exponent length ("up to 16,128-bit long exponents"): 2^16128 mod 2^2048 +- 1
    E = 1 << 16128  # 16129 bits; E mod 2048 = 1792
    assert orc.modexp(2, 16128, (1 << 2048) - 1) == 1 << (16128 % 2048)
    n = (1 << 2048) + 1
    assert orc.modexp(2, 16128, n) == (1 << 1792 if (16128 // 2048) % 2 == 0 else n - (1 << 1792))
    assert E.bit_length() == 16129


def test_modexp_special_values(orc):
    rng = random.Random(5)
    for _ in range(20):
        N = rng.getrandbits(512) | 1 | (1 << 511)
        E = rng.getrandbits(300)
        assert orc.modexp(N - 1, 2 * E, N) == 1
        assert orc.modexp(N - 1, 2 * E + 1, N) == N - 1
        assert orc.modexp(0, E + 1, N) == 0
        assert orc.modexp(0, 0, N) == 1 and orc.modexp(12345, 0, N) == 1
        x = rng.getrandbits(511)
        a, b = rng.getrandbits(100), rng.getrandbits(100)
        assert orc.modexp(x, a + b, N) == orc.modexp(x, a, N) * orc.modexp(x, b, N) % N
    assert orc.modexp(5, 3, 1) == 0


def test_modexp_brute_force_tiny(orc):
    # every x < N, E < 24 for odd N < 2^7 by repeated multiplication (definition of x^E mod N)
    for N in range(3, 128, 2):
        for x in range(N):
            acc = 1 % N
            for E in range(24):
                assert orc.modexp(x, E, N) == acc
                acc = acc * x % N


def test_modexp_vs_cpython_pow(orc):
    rng = random.Random(6)
    for _ in range(400):
        N = rng.getrandbits(rng.randint(2, 1100)) | 1
        x, E = rng.getrandbits(1200), rng.getrandbits(rng.randint(0, 700))
        assert orc.modexp(x, E, N) == pow(x, E, N)


# ---------------------------------------------------------------- O6: inverse

def test_modinv(orc):
    t = load_golden("textbook_rsa.json")
    assert orc.modinv(t["e"], t["phi"]) == t["d"]                # S:86 / S:506: 17^-1 mod 3120 = 2753
    assert orc.modinv(3, 7) == 5                                  # 3*5 = 15 = 1 mod 7
    rng = random.Random(7)
    for _ in range(300):
        m = rng.getrandbits(rng.randint(2, 800)) | 1
        a = rng.getrandbits(800)
        import math
        if math.gcd(a, m) == 1 and m > 1:
            assert orc.modinv(a, m) == pow(a, -1, m)
        elif m > 1:
            with pytest.raises(ValueError):
                orc.modinv(a, m)


# ---------------------------------------------------------------- O7: CRT decryption

def test_crt_toy_worked_example(orc):
    t = load_golden("textbook_rsa.json")
    assert orc.crt_decrypt(t["c"], t["p"], t["q"], t["dp"], t["dq"], t["qinv"], 1) == t["m"]


def test_crt_equals_direct_all_residues_toy(orc):
    # theorem: CRT result = c^d mod n for EVERY c in [0, n), including c sharing a factor with n
    t = load_golden("textbook_rsa.json")
    for c in range(t["n"]):
        assert orc.crt_decrypt(c, t["p"], t["q"], t["dp"], t["dq"], t["qinv"], 1) == pow(c, t["d"], t["n"])


def test_crt_fixture_keys(orc, keys):
    rng = random.Random(8)
    for name in ("rsa1024", "rsa2048"):
        k = keys[name]
        n, p, q = k["n"], k["p"], k["q"]
        nh = (p.bit_length() + 31) // 32
        special = [0, 1, 2, n - 1, p, q, 2 * p, 3 * q]
        for c in special + [rng.randrange(n) for _ in range(6)]:
            m = orc.crt_decrypt(c, p, q, k["dp"], k["dq"], k["qinv"], nh)
            assert m == orc.modexp(c, k["d"], n)                   # CRT-vs-direct agreement
            assert orc.modexp(m, k["e"], n) == c                   # decrypt(encrypt(m)) = m


def test_fixture_keys_are_rsa_keys(keys):
    # invariants of P:54 checked with CPython / sympy (independent of the oracle that made them)
    import sympy
    for name, k in keys.items():
        p, q, e, d = k["p"], k["q"], k["e"], k["d"]
        assert p * q == k["n"] and k["n"].bit_length() == k["bits"]
        assert sympy.isprime(p) and sympy.isprime(q) and p != q
        assert e * d % ((p - 1) * (q - 1)) == 1 and 0 < d < (p - 1) * (q - 1)
        assert k["dp"] == d % (p - 1) and k["dq"] == d % (q - 1) and k["qinv"] * q % p == 1


# ---------------------------------------------------------------- O8 / O9: Miller-Rabin, sieve

def test_small_primes(orc):
    nt = load_golden("number_theory.json")
    ps = orc.small_primes(10000)
    assert ps[:5] == [2, 3, 5, 7, 11] and len(ps) == 10000
    assert ps[-1] == nt["ten_thousandth_prime"]["value"]          # 104729
    assert sum(1 for p in ps if p < 100000) == nt["primes_below_100000"]["count"]


def test_mr_carmichael_rejected(orc):
    import synth
    nt = load_golden("number_theory.json")
    for n in nt["carmichael_below_100000"]["values"]:
        for seed in range(10):
            v, w = orc.miller_rabin(n, synth.mr_bases(n, 20, seed, n))
            assert v == 0 and 0 <= w < 20
    v, w = orc.miller_rabin(561, [2])                              # 2^560 = 1 mod 561, yet strong test fails
    assert (v, w) == (0, 0)


def test_mr_strong_pseudoprimes_round_level(orc):
    nt = load_golden("number_theory.json")["strong_pseudoprimes"]
    for n, bases in nt["values"]:
        assert orc.miller_rabin(n, bases) == (1, -1)               # passes the first primes (A014233)
        nxt = nt["fails_next_base"][str(n)]
        assert orc.miller_rabin(n, bases + [nxt]) == (0, len(bases))   # witness is exactly the next round


def test_mr_completeness_small_primes(orc):
    import synth
    ps = [p for p in orc.small_primes(9592) if p >= 5]
    for i, p in enumerate(ps):
        assert orc.miller_rabin(p, synth.mr_bases(p, 2, 11, i))[0] == 1   # no false composites, ever
    assert orc.miller_rabin(2147483647, [2, 3, 5, 7, 11, 13])[0] == 1     # 2^31 - 1
    assert orc.miller_rabin(9, [2])[0] == 0


def test_mr_mersenne_and_products(orc):
    import synth
    for p in (521, 607, 1279):
        mp = (1 << p) - 1
        assert orc.miller_rabin(mp, synth.mr_bases(mp, 3, 12, p))[0] == 1
    a, b = (1 << 521) - 1, (1 << 607) - 1
    assert orc.miller_rabin(a * b, synth.mr_bases(a * b, 3, 13, 0))[0] == 0


def test_mr_chernick_carmichael(orc):
    # (6t+1)(12t+1)(18t+1) with three prime factors is a Carmichael number of any size: MR says COMPOSITE
    import sympy
    import synth
    t = 1 << 200
    while not (sympy.isprime(6 * t + 1) and sympy.isprime(12 * t + 1) and sympy.isprime(18 * t + 1)):
        t += 1
    n = (6 * t + 1) * (12 * t + 1) * (18 * t + 1)
    assert pow(2, n - 1, n) == 1                                   # a Fermat liar (CPython check)
    assert orc.miller_rabin(n, synth.mr_bases(n, 8, 14, 0))[0] == 0


def test_mr_factor_verdict_and_input_rules(orc):
    bp = orc.base_primes(66)
    assert bp[0] == 4294967291 and bp == sorted(bp, reverse=True)
    n = bp[3] * ((1 << 61) - 1)                                     # > 2^32, divisible by a base prime
    assert orc.miller_rabin(n, [2], bp) == (2, -1)
    assert orc.miller_rabin(n, [2])[0] == 0                         # without the base list: plain MR
    assert orc.miller_rabin(15, [1])[0] == -1                       # base outside [2, n-2]
    assert orc.miller_rabin(16, [2])[0] == -1                       # even n
    assert orc.miller_rabin(3, [2])[0] == -1                        # n < 5


def test_mr_vs_sympy(orc):
    import sympy
    import synth
    for i in range(150):
        n = synth.odd_with_top_bits(256, 21, synth.TAG_CAND, i)
        v, _ = orc.miller_rabin(n, synth.mr_bases(n, 16, 21, i))
        assert (v == 1) == sympy.isprime(n)


@pytest.mark.parametrize("two_k", [20, 130, 194])
def test_base_primes_are_the_largest_primes(orc, two_k):
    """reading R1: the largest primes below 2^32, restricted to primes = 3 mod 4 for k <= 65."""
    import sympy
    bp = orc.base_primes(two_k)
    expect, x = [], 1 << 32
    while len(expect) < two_k:
        x = sympy.prevprime(x)
        if two_k > 130 or x % 4 == 3:
            expect.append(x)
    assert bp == expect


# ---------------------------------------------------------------- O12: threaded drivers = scalar

def test_batch_drivers_match_scalar(orc, keys):
    import numpy as np
    import synth
    k = keys["rsa1024"]
    x = synth.messages(k["n"], 16, 99, 32)
    y = orc.modexp_batch(x, k["e"], k["n"], threads=4)
    for i in range(16):
        xi = int.from_bytes(x[i].tobytes(), "little")
        assert int.from_bytes(y[i].tobytes(), "little") == pow(xi, k["e"], k["n"])
    m = orc.crt_decrypt_batch(y, k["p"], k["q"], k["dp"], k["dq"], k["qinv"], 16, threads=3)
    assert np.array_equal(m, x)
    ns = np.stack([orc.limbs_of(v, 2) for v in (561, 2047, 104729, 1373653)])
    bases = np.stack([np.stack([orc.limbs_of(b, 2) for b in (2, 3)]) for _ in range(4)])
    v, w = orc.miller_rabin_batch(ns, bases, threads=2)
    assert list(v) == [0, 0, 1, 1] and list(w) == [0, 1, -1, -1]
