"""Pins of the DRBG / FIPS 140-2 oracle (oracle/drbg.py; R20-R22).

SHA-256 (hashlib) is pinned to the FIPS 180-2 example digests; the FIPS 140-2 thresholds are pinned to
their binomial / chi-square tail probabilities (the standard's ~1e-4 two-sided bands) and the expected
run counts; every statistic is pinned on constructed blocks whose values follow by hand (all zeros,
alternating bits, exact ones counts at the monobit edges, a run of exactly 25 / 26, chosen nibble
histograms at the poker edges).  Hash_DRBG itself has no offline SP 800-90A vector here: its pins are the
structural properties (determinism, domain separation of streams, the mod 2^440 counter wrap, the
reseed-counter update); its values are pinned against OpenSSL 3's HASH-DRBG in
tests/test_oracle_standard_pins.py."""
import numpy as np
import pytest

from oracle import drbg


def test_sha256_fips180_examples():
    assert drbg.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    msg = b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq"
    assert drbg.sha256(msg).hex() == "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"


def test_thresholds_are_the_standard_tail_bands():
    from scipy.stats import binom, chi2
    lo, hi = drbg.MONOBIT
    assert 3e-5 < binom.cdf(lo, 20000, 0.5) < 1e-4 and 3e-5 < binom.sf(hi - 1, 20000, 0.5) < 1e-4
    assert 3e-5 < chi2.cdf(drbg.POKER_X[0], 15) < 1e-4 and 3e-5 < chi2.sf(drbg.POKER_X[1], 15) < 1e-4
    for ln, (a, b) in enumerate(drbg.RUNS[:5], start=1):
        e = (20000 - ln + 3) / 2 ** (ln + 2)            # expected runs of one bit value, exact length ln
        assert a < e < b and abs((a + b) / 2 - e) < 2
    e6 = sum((20000 - ln + 3) / 2 ** (ln + 2) for ln in range(6, 20000))
    assert drbg.RUNS[5][0] < e6 < drbg.RUNS[5][1]


def _block_from_bits(bits):
    return np.packbits(np.asarray(bits, dtype=np.uint8)).tobytes()


def test_health_all_zeros_and_alternating():
    z = drbg.health(bytes(2500))
    assert z["ones"] == 0 and z["longest"] == 20000 and not z["monobit"] and not z["long_run"]
    assert z["poker_s"] == 5000 ** 2 and not z["poker"] and z["runs"][0, 5] == 1 and z["runs"].sum() == 1
    a = drbg.health(bytes([0x55]) * 2500)
    assert a["ones"] == 10000 and a["monobit"] and a["longest"] == 1 and a["long_run"]
    assert a["runs"][0, 0] == 10000 and a["runs"][1, 0] == 10000 and not a["runs_ok"]
    assert not a["poker"]                                            # every nibble is 0x5


def test_health_monobit_edges_and_long_run():
    rng = np.random.default_rng(5)
    for ones, ok in ((9725, False), (9726, True), (10274, True), (10275, False)):
        bits = np.zeros(20000, dtype=np.uint8)
        bits[rng.choice(20000, ones, replace=False)] = 1
        h = drbg.health(_block_from_bits(bits))
        assert h["ones"] == ones and h["monobit"] == ok
    for ln, ok in ((25, True), (26, False)):
        bits = np.tile(np.array([0, 1], dtype=np.uint8), 10000)
        bits[1000:1000 + ln] = 1
        bits[1000 - 1] = 0
        bits[1000 + ln] = 0
        h = drbg.health(_block_from_bits(bits))
        assert h["longest"] == ln and h["long_run"] == ok


def test_health_poker_edges():
    # nibble histograms with S = sum f^2 just inside / outside 1,563,175 < S < 1,576,928
    def block_with_counts(f):
        nib = np.repeat(np.arange(16, dtype=np.uint8), f)
        np.random.default_rng(1).shuffle(nib)
        return (nib[0::2] << 4 | nib[1::2]).astype(np.uint8).tobytes()
    base = np.full(16, 312)
    base[:8] += 1                                                    # 8 x 313 + 8 x 312 = 5000
    assert base.sum() == 5000
    f = base.copy()
    s = int((f ** 2).sum())
    h = drbg.health(block_with_counts(f))
    assert h["poker_s"] == s and not h["poker"]                      # S = 1,562,504: X = 0.01 < 2.16
    # move counts between two cells until S crosses the lower edge
    while int((f ** 2).sum()) <= 1563175:
        f[0] += 1
        f[15] -= 1
    h = drbg.health(block_with_counts(f))
    assert h["poker_s"] == int((f ** 2).sum()) and h["poker"]


def test_hash_drbg_structure():
    e, n = bytes(range(32)), bytes(range(16))
    a, b = drbg.HashDrbg(e, n, b"x"), drbg.HashDrbg(e, n, b"x")
    assert a.generate(100) == b.generate(100) and a.reseed_counter == 2
    c = drbg.HashDrbg(e, n, b"y")
    assert c.generate(64) != drbg.HashDrbg(e, n, b"x").generate(64)     # personalization separates streams
    s0, s1 = drbg.generate_batch(e, n, b"p", 2, 64)[0]
    assert not np.array_equal(s0, s1)
    # Hashgen is counter mode over V (mod 2^440): the block after V = 2^440 - 1 is the hash of V = 0
    d = drbg.HashDrbg(e, n, b"")
    d.V = (1 << 440) - 1
    out = d.hashgen(64)
    assert out[32:] == drbg.sha256(bytes(55))
    with pytest.raises(ValueError):
        d.generate(drbg.MAX_REQUEST_BYTES + 1)


def test_drbg_output_passes_health():
    d = drbg.HashDrbg(b"\x01" * 32, b"\x02" * 16, b"health")
    data = d.hashgen(2500 * 100)
    passed = sum(all(drbg.health(data[i * 2500:(i + 1) * 2500])[k] for k in ("monobit", "poker", "runs_ok", "long_run"))
                 for i in range(100))
    assert passed >= 98
