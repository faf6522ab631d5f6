"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element on the same
seeded inputs.  Bit-exact: every output is an integer with a unique value.

Covers C1 in full (RSA-1024: 256 messages, encrypt e = 65537, decrypt with the full d, and CRT
decrypt), tiny moduli by brute force (k = 1), random exponents, ragged batch sizes spanning several
CTAs, edge inputs, out-of-range status, prefix determinism, long exponents with closed forms, and
the full-size C2 launch on sampled outputs.
"""
import random

import numpy as np
import pytest

import synth
from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def mr():
    import paper_1305_3699_b200 as mr
    mr.lib()
    return mr


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def ints(a):
    return [int.from_bytes(np.ascontiguousarray(r).tobytes(), "little") for r in np.asarray(a, dtype=np.uint32)]


def run_modexp(torch, mr, N, xs, E, limbs=None, k=0):
    limbs = limbs or (N.bit_length() + 31) // 32
    ctx = mr.RnsContext(N, limbs, k=k)
    x = dev(torch, mr.ints_to_limbs(xs, limbs))
    y = torch.empty_like(x)
    st = torch.zeros(len(xs), dtype=torch.int32, device="cuda")
    ctx.modexp(x, y, E, d_status=st)
    torch.cuda.synchronize()
    return ints(host(y)), host(st).view(np.int32).tolist(), ctx


def test_textbook_rsa(torch_cuda, mr):
    t = load_golden("textbook_rsa.json")
    y, st, ctx = run_modexp(torch_cuda, mr, t["n"], [t["m"]], t["e"])
    assert ctx.k == 1 and y == [t["c"]] and st == [0]                     # 65^17 mod 3233 = 2790
    y, _, _ = run_modexp(torch_cuda, mr, t["n"], [t["c"]], t["d"])
    assert y == [t["m"]]                                                  # 2790^2753 mod 3233 = 65
    key = mr.RsaPrivateKey(t["p"], t["q"], t["dp"], t["dq"], t["qinv"], half_limbs=1)
    c = dev(torch_cuda, mr.ints_to_limbs(list(range(t["n"])), 2))
    m = torch_cuda.empty_like(c)
    key.decrypt(c, m)
    torch_cuda.cuda.synchronize() if hasattr(torch_cuda, "cuda") else None
    assert ints(host(m)) == [pow(v, t["d"], t["n"]) for v in range(t["n"])]   # CRT for every c < n


def test_brute_force_tiny_moduli(torch_cuda, mr, orc):
    # every x < N, E in a spread of small exponents, for a set of odd N (k = 1)
    rng = random.Random(1)
    for N in [3, 5, 7, 9, 15, 255, 257, 1001, 3233, 4095, 65535, 65537, (1 << 20) + 7]:
        xs = list(range(N)) if N < 5000 else [rng.randrange(N) for _ in range(3000)]
        for E in (0, 1, 2, 3, 5, 17, 64, 65537, rng.getrandbits(40)):
            y, st, _ = run_modexp(torch_cuda, mr, N, xs, E)
            assert y == [orc.modexp(x, E, N) for x in xs], (N, E)
            assert all(s == 0 for s in st)


@pytest.mark.parametrize("bits", [64, 256, 512, 1000, 1024, 1536, 2048, 3072, 4000])
def test_random_moduli_and_exponents(torch_cuda, mr, orc, bits):
    rng = random.Random(bits)
    N = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
    count = 257                                                          # ragged: 3 CTAs of 128
    xs = [rng.randrange(N) for _ in range(count)]
    for E in (65537, rng.getrandbits(bits), rng.getrandbits(97) | 1):
        y, st, _ = run_modexp(torch_cuda, mr, N, xs, E)
        expect = orc.modexp_batch(mr.ints_to_limbs(xs, (bits + 31) // 32), E, N, threads=8)
        assert y == ints(expect)


def test_c1_full(torch_cuda, mr, orc, keys):
    """C1: RSA-1024, 256 seeded messages, encrypt e=65537, decrypt with the full d (non-CRT) and CRT."""
    k = keys["rsa1024"]
    n, L = k["n"], 32
    msgs = synth.messages(n, 256, 0x5EEDC001, L, edge=synth.edge_values(n, k["p"], k["q"]))
    c_ref = orc.modexp_batch(msgs, k["e"], n, threads=8)
    ctx = mr.RnsContext(n, L)
    assert ctx.k == 33
    x = dev(torch_cuda, msgs)
    c = torch_cuda.empty_like(x)
    ctx.encrypt(x, c, k["e"])
    m1 = torch_cuda.empty_like(x)
    ctx.modexp(c, m1, k["d"])
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    m2 = torch_cuda.empty_like(x)
    key.decrypt(c, m2)
    torch_cuda.cuda.synchronize()
    assert np.array_equal(host(c), c_ref)                                 # encrypt == oracle, all 256
    assert np.array_equal(host(m1), msgs)                                 # decrypt(encrypt(m)) = m
    assert np.array_equal(host(m2), msgs)                                 # CRT decrypt = m
    d_ref = orc.modexp_batch(c_ref[:64], k["d"], n, threads=8)
    assert np.array_equal(host(m1)[:64], d_ref)                           # decrypt == oracle


def test_crt_decrypt_rsa2048_edges(torch_cuda, mr, orc, keys):
    k = keys["rsa2048"]
    n, p, q = k["n"], k["p"], k["q"]
    edge = [0, 1, 2, n - 1, n - 2, p, q, 2 * p, 3 * q, p * 5, q - 1, p + 1, 0xDEADBEEF]
    cs = synth.messages(n, 300, 77, 64, edge=edge)
    key = mr.RsaPrivateKey(p, q, k["dp"], k["dq"], k["qinv"])
    c = dev(torch_cuda, cs)
    m = torch_cuda.empty_like(c)
    st = torch_cuda.zeros(300, dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=st)
    torch_cuda.cuda.synchronize()
    ref = orc.crt_decrypt_batch(cs, p, q, k["dp"], k["dq"], k["qinv"], 32, threads=8)
    assert np.array_equal(host(m), ref)
    assert (host(st) == 0).all()


def test_out_of_range_status(torch_cuda, mr, keys):
    k = keys["rsa1024"]
    n = k["n"]
    xs = [5, n, n + 1, (1 << 1024) - 1, n - 1]
    y, st, _ = run_modexp(torch_cuda, mr, n, xs, k["e"])
    assert st == [0, 5, 5, 5, 0]
    assert y[1] == y[2] == y[3] == 0 and y[0] == pow(5, k["e"], n) and y[4] == n - 1
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    c = dev(torch_cuda, mr.ints_to_limbs([n, 7], 32))
    m = torch_cuda.empty_like(c)
    s2 = torch_cuda.zeros(2, dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=s2)
    torch_cuda.cuda.synchronize()
    assert host(s2).view(np.int32).tolist() == [5, 0] and ints(host(m)) == [0, pow(7, k["d"], n)]


def test_batch_size_determinism(torch_cuda, mr, keys):
    """prefix property: the first n outputs of a 2n batch equal an n batch (any tile split)."""
    k = keys["rsa1024"]
    n = k["n"]
    msgs = synth.messages(n, 1000, 5, 32)
    outs = {}
    for cnt in (1, 127, 128, 129, 1000):
        y, _, _ = run_modexp(torch_cuda, mr, n, ints(msgs[:cnt]), k["d"])
        outs[cnt] = y
    for cnt in (1, 127, 128, 129):
        assert outs[cnt] == outs[1000][:cnt]


def test_empty_batch(torch_cuda, mr, keys):
    ctx = mr.RnsContext(keys["rsa1024"]["n"])
    x = torch_cuda.zeros((0, 32), dtype=torch_cuda.int32, device="cuda")
    ctx.modexp(x, x, 65537)


@pytest.mark.parametrize("ell", [17, 1024, 4096, 16128])
def test_long_exponent_closed_forms(torch_cuda, mr, ell):
    """C4 shape: 2^E mod (2^2048 +- 1) in closed form, E up to 16,128 bits."""
    E = synth.exponent(ell, 0x5EEDC004)
    for N in ((1 << 2048) - 1, (1 << 2048) + 1):
        limbs = (N.bit_length() + 31) // 32
        y, _, ctx = run_modexp(torch_cuda, mr, N, [2, 1, N - 1], E, limbs=limbs)
        r = 1 << (E % 2048)
        if N == (1 << 2048) - 1:
            assert y[0] == r
        else:
            assert y[0] == (r if (E // 2048) % 2 == 0 else N - r)
        assert y[1] == 1 and y[2] == (1 if E % 2 == 0 else N - 1)


def test_c4_sampled_vs_oracle(torch_cuda, mr, orc, keys):
    k = keys["rsa2048"]
    n = k["n"]
    E = synth.exponent(4096, 0x5EEDC004, 1)
    xs = synth.messages(n, 64, 0x5EEDC004, 64)
    y, _, ctx = run_modexp(torch_cuda, mr, n, ints(xs), E)
    assert ctx.k == 65
    assert y == ints(orc.modexp_batch(xs, E, n, threads=8))


def test_c2_full_size_sampled(torch_cuda, mr, orc, keys):
    """C2 at BASELINE size (65,536 RSA-2048 CRT decryptions, the bench launch) on sampled outputs,
    plus the property enc(dec(c)) = c on all of them (computed on the GPU, encrypt is itself
    parity-tested above)."""
    k = keys["rsa2048"]
    n, count = k["n"], 65536
    cs = synth.messages(n, count, 0x5EEDC002, 64, edge=synth.edge_values(n, k["p"], k["q"]))
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    ctx = mr.RnsContext(n)
    c = dev(torch_cuda, cs)
    m = torch_cuda.empty_like(c)
    key.decrypt(c, m)
    c2 = torch_cuda.empty_like(c)
    ctx.encrypt(m, c2, k["e"])
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(c, c2)
    idx = list(range(0, 512)) + list(range(512, count, 257))
    ref = orc.crt_decrypt_batch(cs[idx], k["p"], k["q"], k["dp"], k["dq"], k["qinv"], 32, threads=8)
    assert np.array_equal(host(m)[idx], ref)


def test_c3_rsa3072_encrypt_decrypt(torch_cuda, mr, orc, keys):
    """C3 shape: RSA-3072 encryption (k = 97) and CRT decryption (k = 49 per half), ragged batch."""
    k = keys["rsa3072"]
    n, L = k["n"], 96
    msgs = synth.messages(n, 300, 0x5EEDC003, L, edge=synth.edge_values(n, k["p"], k["q"]))
    ctx = mr.RnsContext(n, L)
    assert ctx.k == 97
    x = dev(torch_cuda, msgs)
    c = torch_cuda.empty_like(x)
    ctx.encrypt(x, c, k["e"])
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    m = torch_cuda.empty_like(x)
    key.decrypt(c, m)
    torch_cuda.cuda.synchronize()
    ref = orc.modexp_batch(msgs[:96], k["e"], n, threads=8)
    assert np.array_equal(host(c)[:96], ref)
    assert np.array_equal(host(m), msgs)


def test_k65_pair_path_ragged(torch_cuda, mr, orc, keys):
    """k = 65 (2048-bit N, CTA-pair tensor kernel): a ragged batch over several
    256-message pair jobs, every output vs the oracle, for e = 65537 and for the full d."""
    k = keys["rsa2048"]
    n = k["n"]
    xs = synth.messages(n, 1000, 0x5EEDC065, 64, edge=synth.edge_values(n, k["p"], k["q"]))
    y, st, ctx = run_modexp(torch_cuda, mr, n, ints(xs), k["e"])
    assert ctx.k == 65 and st == [0] * 1000
    assert y == ints(orc.modexp_batch(xs, k["e"], n, threads=8))
    sub = xs[:300]
    yd, _, _ = run_modexp(torch_cuda, mr, n, ints(sub), k["d"])
    assert yd == ints(orc.modexp_batch(sub, k["d"], n, threads=8))


def test_c4_full_size_round_trip(torch_cuda, mr, orc, keys):
    """C4 launch size (65,536 messages over a 2048-bit N, k = 65): (x^d)^e = x for every message
    (both legs on the GPU; the e leg is oracle-checked above) and x^d vs the oracle on a sample."""
    k = keys["rsa2048"]
    n, count = k["n"], 65536
    xs = synth.messages(n, count, 0x5EEDC004, 64, edge=synth.edge_values(n, k["p"], k["q"]))
    ctx = mr.RnsContext(n)
    assert ctx.k == 65
    x = dev(torch_cuda, xs)
    y = torch_cuda.empty_like(x)
    z = torch_cuda.empty_like(x)
    ctx.modexp(x, y, k["d"])
    ctx.modexp(y, z, k["e"])
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(x, z)
    idx = list(range(0, 96)) + list(range(96, count, 1021))
    assert np.array_equal(host(y)[idx], orc.modexp_batch(xs[idx], k["d"], n, threads=8))


@pytest.mark.parametrize("bits", [3072, 4096, 8192, 16128])
def test_wide_moduli_vs_oracle(torch_cuda, mr, orc, bits):
    """§8(f) row 3, wide operands (k = 97 / 129 / 257 / 505, channels-on-threads kernel): a ragged batch
    of 37 messages (three 16-message CTAs) for e = 65537 and a 300-bit exponent, every output vs the oracle,
    with edge inputs 0, 1, N-1 and one out-of-range input."""
    rng = random.Random(bits)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    limbs = (bits + 31) // 32
    xs = [0, 1, N - 1] + [rng.randrange(N) for _ in range(33)] + [N + 5]
    for E in (65537, rng.getrandbits(300) | (1 << 299)):
        y, st, ctx = run_modexp(torch_cuda, mr, N, xs, E, limbs=limbs)
        assert ctx.k == {3072: 97, 4096: 129, 8192: 257, 16128: 505}[bits]
        assert st == [0] * 36 + [5] and y[36] == 0
        ref = ints(orc.modexp_batch(mr.ints_to_limbs(xs[:36], limbs), E, N, threads=8))
        assert y[:36] == ref


@pytest.mark.parametrize("n", [4000, 8192, 16128])
def test_wide_closed_forms(torch_cuda, mr, n):
    """2^E mod (2^n + 1) = ±2^(E mod n) for a 16,128-bit exponent (the paper's long-exponent shape)."""
    E = synth.exponent(16128, 0x5EEDC0DE)
    N = (1 << n) + 1
    limbs = (N.bit_length() + 31) // 32
    y, _, ctx = run_modexp(torch_cuda, mr, N, [2, 1, N - 1], E, limbs=limbs)
    r = 1 << (E % n)
    assert y[0] == (r if (E // n) % 2 == 0 else N - r)
    assert y[1] == 1 and y[2] == (1 if E % 2 == 0 else N - 1)


def test_wide_crt_decrypt_vs_oracle(torch_cuda, mr, orc):
    """CRT decryption with 8064-bit halves (a 16,128-bit key shape; halves on the wide kernel with the
    positional recombination).  Garner's recombination (O7) is defined for any coprime odd p, q and any
    d_p, d_q, so random ones serve (no 8064-bit prime search on the CPU); every output vs the oracle,
    ragged batch of 21 with edge inputs and one out-of-range ciphertext."""
    import math
    rng = random.Random(16128)
    while True:
        p = rng.getrandbits(8064) | (3 << 8062) | 1
        q = rng.getrandbits(8064) | (3 << 8062) | 1
        if p != q and math.gcd(p, q) == 1:
            break
    n, H = p * q, 252
    dp, dq = rng.getrandbits(96) | 1, rng.getrandbits(96) | 1
    qinv = pow(q, -1, p)
    cs = [0, 1, n - 1, p, q] + [rng.randrange(n) for _ in range(15)] + [n + 3]
    key = mr.RsaPrivateKey(p, q, dp, dq, qinv)
    c = dev(torch_cuda, mr.ints_to_limbs(cs, 2 * H))
    m = torch_cuda.empty_like(c)
    st = torch_cuda.zeros(len(cs), dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=st)
    torch_cuda.cuda.synchronize()
    assert host(st).view(np.int32).tolist() == [0] * 20 + [5]
    got = host(m)
    ref = orc.crt_decrypt_batch(mr.ints_to_limbs(cs[:20], 2 * H), p, q, dp, dq, qinv, H, threads=8)
    assert np.array_equal(got[:20], ref) and not got[20].any()


@pytest.mark.parametrize("count", [37889, 38016, 75777])
def test_split_schedule_geometries(torch_cuda, mr, orc, keys, count):
    """the wrap-around schedule of DESIGN.md §4f at awkward job counts: CRT decryption with 297 and
    297 (ragged) tile-jobs per context on 296 slots (one job straddles two slots), and encryption-then-
    decryption round trips; sampled outputs vs the oracle, every output by the round trip."""
    k = keys["rsa2048"]
    n = k["n"]
    cs = synth.messages(n, count, 0x5EEDC0C0 + count, 64)
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    ctx = mr.RnsContext(n)
    c = dev(torch_cuda, cs)
    m = torch_cuda.empty_like(c)
    key.decrypt(c, m)
    c2 = torch_cuda.empty_like(c)
    ctx.encrypt(m, c2, k["e"])
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(c, c2)
    idx = [0, 1, 127, 128, count // 2, count - 129, count - 2, count - 1]
    ref = orc.crt_decrypt_batch(cs[idx], k["p"], k["q"], k["dp"], k["dq"], k["qinv"], 32, threads=8)
    assert np.array_equal(host(m)[idx], ref)


@pytest.mark.parametrize("half_bits", [2048, 4096])
def test_crt_decrypt_large_halves_vs_oracle(torch_cuda, mr, orc, half_bits):
    """CRT decryption with 2048-bit halves (k = 65: both contexts on the CTA-pair tensor kernel in one
    launch) and 4096-bit halves (k = 129, wide-operand kernel, positional recombination): random coprime odd p, q (Garner's definition O7 needs
    no primality), ragged batch of 300 with edge inputs, every output vs the oracle."""
    import math
    rng = random.Random(half_bits)
    while True:
        p = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        q = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        if p != q and math.gcd(p, q) == 1:
            break
    n, H = p * q, half_bits // 32
    dp, dq = rng.getrandbits(128) | 1, rng.getrandbits(128) | 1
    qinv = pow(q, -1, p)
    cs = [0, 1, n - 1, p, q, 2 * p] + [rng.randrange(n) for _ in range(294)]
    key = mr.RsaPrivateKey(p, q, dp, dq, qinv)
    c = dev(torch_cuda, mr.ints_to_limbs(cs, 2 * H))
    m = torch_cuda.empty_like(c)
    key.decrypt(c, m)
    torch_cuda.cuda.synchronize()
    ref = orc.crt_decrypt_batch(mr.ints_to_limbs(cs, 2 * H), p, q, dp, dq, qinv, H, threads=8)
    assert np.array_equal(host(m), ref)


_PER_K_SNIPPET = r"""
import random, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1305_3699_b200 as mr
for bits in (3072, 4096):
    rng = random.Random(bits + 1)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [0, 1, N - 1] + [rng.randrange(N) for _ in range(130)]
    E = rng.getrandbits(200) | (1 << 199)
    ctx = mr.RnsContext(N, L)
    x = torch.from_numpy(mr.ints_to_limbs(xs, L).view(np.int32)).cuda()
    y = torch.empty_like(x)
    ctx.modexp(x, y, E)
    got = mr.limbs_to_ints(y.cpu().numpy())
    assert got == [pow(v, E, N) for v in xs], bits
print("per-k ok")
"""


def test_per_k_imad_modexp_k97_k129(torch_cuda):
    """The per-k IMAD modexp kernels of k = 97 / 129 are no longer the default (the wide kernel runs those
    sizes) but stay selectable (MR_RNS_WIDE_MIN=999, read once per process): a subprocess
    runs 133 messages (ragged over 64/128-message CTAs, edges 0, 1, N-1) per size against Python's pow."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MR_RNS_WIDE_MIN="999")
    r = subprocess.run([sys.executable, "-c", _PER_K_SNIPPET.format(root=root)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "per-k ok" in r.stdout, r.stderr[-2000:]
