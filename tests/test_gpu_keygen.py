"""GPU RSA key generation (mr_rsa_keygen_batch) against the oracle recipe.

Expected keys come from scripts/gen_fixtures.gen_key, which calls only oracle/ (next_prime with
trial division + Miller-Rabin, modinv, divmod) and synth/ (seeded starts): the committed fixtures
tests/golden/keys/*.json are key 0 of that recipe (reading R19), so the GPU must reproduce them
limb for limb.  Larger batches are checked on sampled keys against the recipe and, for every key,
against properties that define an RSA key (n = p q, e d = 1 mod lcm, q q_inv = 1 mod p, d_p, d_q).
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, load_key

sys.path.insert(0, os.path.join(ROOT, "scripts"))

FIELDS = ("n", "p", "q", "d", "dp", "dq", "qinv")


def _mr():
    import paper_1305_3699_b200 as mr
    return mr


def keygen(count, bits, e, seed, rounds, first_key=0):
    import torch
    mr = _mr()
    full, half = bits // 32, bits // 64
    out = {f: torch.zeros((max(count, 1), full if f in ("n", "d") else half), dtype=torch.int32, device="cuda")
           for f in FIELDS}
    mr.mr_rsa_keygen_batch(count, bits, e, seed, rounds, out["n"], out["p"], out["q"], out["d"], out["dp"],
                           out["dq"], out["qinv"], first_key=first_key)
    torch.cuda.synchronize()
    res = []
    host = {f: out[f].cpu().numpy().view(np.uint32) for f in FIELDS}
    for i in range(count):
        res.append({f: int.from_bytes(host[f][i].tobytes(), "little") for f in FIELDS})
    return res


def test_keygen_rejects_bad_arguments():
    """argument validation happens before any device work (runs on CPU too)."""
    mr = _mr()
    L = mr.lib()
    for bits, e, rounds in ((1000, 65537, 8), (128, 65537, 8), (1024, 65536, 8), (1024, 65537, 0), (1024, 1, 8),
                            (8192, 65537, 8), (1024, 65537 * 3, 8)):
        assert L.mr_rsa_keygen_batch(1, bits, e, 1, 0, rounds, *([None] * 7), 0, None) == mr.MR_ERR_ARG
    assert L.mr_rsa_keygen_batch(0, 1024, 65537, 1, 0, 8, *([None] * 7), 0, None) == mr.MR_OK


@pytest.mark.gpu
@pytest.mark.parametrize("name,bits,seed", [("rsa1024", 1024, 0x5EEDC001), ("rsa2048", 2048, 0x5EEDC002),
                                            ("rsa3072", 3072, 0x5EEDC003)])
def test_keygen_reproduces_committed_fixtures(name, bits, seed):
    """key 0 of the recipe with 64 MR rounds = the committed oracle fixture, every field."""
    ref = load_key(name)
    got = keygen(1, bits, 65537, seed, 64)[0]
    for f in FIELDS:
        assert got[f] == ref[f], f


@pytest.mark.gpu
def test_keygen_batch_matches_oracle_recipe(orc):
    """8 keys at key indices 5..12, 10 rounds, e = 3 (gcd(e, p-1) rejections are frequent: 1/2 of primes)."""
    import gen_fixtures
    got = keygen(8, 1024, 3, 0xC0FFEE, 10, first_key=5)
    for i, g in enumerate(got):
        ref = gen_fixtures.gen_key(1024, 0xC0FFEE, key_index=5 + i, rounds=10, e=3)
        for f in FIELDS:
            assert g[f] == int(ref[f], 16), (i, f)


@pytest.mark.gpu
def test_keygen_index_stability():
    """a key depends only on (seed, global key index): batch [0, 6) and batch [2, 4) agree."""
    a = keygen(6, 512, 65537, 77, 6)
    b = keygen(2, 512, 65537, 77, 6, first_key=2)
    assert a[2:4] == b


@pytest.mark.gpu
def test_keygen_batch_properties_and_sample(orc):
    """256 RSA-2048 keys, 5 rounds: every key is a valid RSA key; 2 sampled keys equal the recipe;
    p and q of 16 keys pass 20 oracle MR rounds with random bases."""
    import random
    import gen_fixtures
    e = 65537
    got = keygen(256, 2048, e, 0xABCDEF, 5)
    for g in got:
        p, q = g["p"], g["q"]
        assert g["n"] == p * q and g["n"].bit_length() == 2048
        assert p.bit_length() == q.bit_length() == 1024 and p >> 1022 == 3 and q >> 1022 == 3
        assert abs(p - q).bit_length() > 1024 - 100
        phi = (p - 1) * (q - 1)
        assert g["d"] * e % phi == 1 and 0 < g["d"] < phi
        assert g["dp"] == g["d"] % (p - 1) and g["dq"] == g["d"] % (q - 1)
        assert g["qinv"] * q % p == 1 and 0 < g["qinv"] < p
    assert len({g["n"] for g in got}) == 256
    for i in (0, 255):
        ref = gen_fixtures.gen_key(2048, 0xABCDEF, key_index=i, rounds=5, e=e)
        for f in FIELDS:
            assert got[i][f] == int(ref[f], 16), (i, f)
    rng = random.Random(5)
    fp = orc.base_primes(66)
    for g in got[:16]:
        for x in (g["p"], g["q"]):
            v, _ = orc.miller_rabin(x, [rng.randrange(2, x - 1) for _ in range(20)], fp)
            assert v == orc.PROBABLY_PRIME


def keygen_drbg(count, bits, e, rounds, entropy, nonce=b"\x00" * 16, streams=64):
    import torch
    mr = _mr()
    rng = mr.Drbg(entropy, nonce, b"keygen", streams=streams)
    full, half = bits // 32, bits // 64
    out = {f: torch.zeros((count, full if f in ("n", "d") else half), dtype=torch.int32, device="cuda")
           for f in FIELDS}
    mr.mr_rsa_keygen_batch_drbg(rng, count, bits, e, rounds, out["n"], out["p"], out["q"], out["d"], out["dp"],
                                out["dq"], out["qinv"])
    torch.cuda.synchronize()
    host = {f: out[f].cpu().numpy().view(np.uint32) for f in FIELDS}
    return [{f: int.from_bytes(host[f][i].tobytes(), "little") for f in FIELDS} for i in range(count)]


@pytest.mark.gpu
def test_keygen_drbg_valid_keys_and_determinism(orc):
    """the production entry draws starts and every Miller-Rabin base from the GPU
    Hash_DRBG.  Every key is a valid RSA key whose primes pass 20 oracle MR rounds and sympy's BPSW; the
    same entropy gives the same keys, other entropy other keys; the keys differ from the seeded recipe."""
    import random
    import sympy
    e = 65537
    ent = bytes(range(32))
    got = keygen_drbg(64, 2048, e, 5, ent)
    for g in got:
        p, q = g["p"], g["q"]
        assert g["n"] == p * q and g["n"].bit_length() == 2048
        assert p >> 1022 == 3 and q >> 1022 == 3 and abs(p - q).bit_length() > 1024 - 100
        phi = (p - 1) * (q - 1)
        assert g["d"] * e % phi == 1 and g["dp"] == g["d"] % (p - 1) and g["dq"] == g["d"] % (q - 1)
        assert g["qinv"] * q % p == 1
    rng = random.Random(9)
    fp = orc.base_primes(66)
    for g in got[:8]:
        for x in (g["p"], g["q"]):
            assert sympy.isprime(x)
            v, _ = orc.miller_rabin(x, [rng.randrange(2, x - 1) for _ in range(20)], fp)
            assert v == orc.PROBABLY_PRIME
    assert len({g["p"] for g in got} | {g["q"] for g in got}) == 128
    assert keygen_drbg(64, 2048, e, 5, ent) == got      # same entropy and request pattern: same keys
    other = keygen_drbg(8, 2048, e, 5, bytes(range(1, 33)))
    assert not ({o["n"] for o in other} & {g["n"] for g in got})
    seeded = keygen(1, 2048, e, 0, 5)[0]
    assert seeded["n"] not in {g["n"] for g in got}


@pytest.mark.gpu
def test_keygen_drbg_random_bases_reject_composites():
    """RSA-1024 keys with a single Miller-Rabin round per prime (random base): the primes must still be
    prime with overwhelming probability (a composite that survives sieving passes one random round with
    probability <= 1/4 and typically ~2^-40); checked by sympy for all 32 keys."""
    import sympy
    got = keygen_drbg(32, 1024, 65537, 1, b"\x5a" * 32, streams=8)
    for g in got:
        assert sympy.isprime(g["p"]) and sympy.isprime(g["q"])
