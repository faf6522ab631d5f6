"""GPU parity of mr_miller_rabin_batch (§3.2, HAC 4.24) against the oracle: verdict and first
witnessing round must be identical for the same candidates and the same explicit bases (reading
R13), including the FACTOR verdict of reading R14 and the input rules of include/mr_rns.h."""
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


def gpu_mr(torch, mr, ns, bases, limbs=None):
    """ns: list of ints; bases: list of lists (rounds each). Returns (verdict, witness, status)."""
    limbs = limbs or max(1, max((n.bit_length() + 31) // 32 for n in ns))
    rounds = len(bases[0])
    n_arr = mr.ints_to_limbs(ns, limbs)
    b_arr = np.stack([mr.ints_to_limbs(b, limbs) for b in bases]).reshape(len(ns), rounds, limbs)
    d_n = torch.from_numpy(n_arr.view(np.int32)).cuda()
    d_b = torch.from_numpy(np.ascontiguousarray(b_arr).view(np.int32)).cuda()
    v = torch.zeros(len(ns), dtype=torch.uint8, device="cuda")
    w = torch.zeros(len(ns), dtype=torch.int16, device="cuda")
    s = torch.zeros(len(ns), dtype=torch.int32, device="cuda")
    mr.mr_miller_rabin_batch(d_n, limbs, len(ns), d_b, rounds, v, w, s)
    torch.cuda.synchronize()
    return v.cpu().numpy().tolist(), w.cpu().numpy().tolist(), s.cpu().numpy().tolist(), limbs


def oracle_mr(orc, ns, bases, limbs, k):
    fp = orc.base_primes(2 * k)
    out = []
    for n, b in zip(ns, bases):
        v, w = orc.miller_rabin(n, b, fp)
        out.append((v, w))
    return [v for v, _ in out], [w for _, w in out]


def k_for(mr, limbs):
    for k in mr.mr_rns_supported_k():
        if 4 * (k + 3) ** 2 * (1 << (32 * limbs)) < _M(k) and limbs <= k - 1:
            return k


_MC = {}


def _M(k):
    if k not in _MC:
        import sympy
        ps, x = [], 1 << 32
        while len(ps) < k:
            x = sympy.prevprime(x)
            ps.append(x)
        m = 1
        for p in ps:
            m *= p
        _MC[k] = m
    return _MC[k]


def check(torch, mr, orc, ns, bases):
    v, w, s, limbs = gpu_mr(torch, mr, ns, bases)
    ov, ow = oracle_mr(orc, ns, bases, limbs, k_for(mr, limbs))
    assert v == ov, [(n, a, b) for n, a, b in zip(ns, v, ov) if a != b][:5]
    assert w == ow
    assert all(x == 0 for x in s)
    return v, w


def test_carmichael_and_small_primes(torch_cuda, mr, orc):
    nt = load_golden("number_theory.json")
    car = nt["carmichael_below_100000"]["values"]
    ns = car + [p for p in orc.small_primes(2000) if p >= 5][:500] + [2147483647, 9, 25, 49, 15, 21]
    bases = [synth.mr_bases(n, 20, 3, i) for i, n in enumerate(ns)]
    v, w = check(torch_cuda, mr, orc, ns, bases)
    assert all(x == 0 for x in v[: len(car)])                          # every Carmichael number rejected
    assert all(x == 1 for x in v[len(car): len(car) + 501])            # no false composites


def test_strong_pseudoprimes_round_level(torch_cuda, mr, orc):
    nt = load_golden("number_theory.json")["strong_pseudoprimes"]
    ns, bases = [], []
    for n, bs in nt["values"]:
        ns.append(n)
        bases.append(bs + [nt["fails_next_base"][str(n)]] + [2] * (6 - len(bs)))
    v, w = check(torch_cuda, mr, orc, ns, bases)
    assert v == [0] * len(ns)
    assert w == [len(b) for b, _ in [(bs, 0) for _, bs in nt["values"]]]


def test_c5_shape_1024_bit_candidates(torch_cuda, mr, orc):
    """C5: seeded 1024-bit candidates (top two bits + low bit set), 5 rounds of bases in [2, n-2]."""
    ns = [synth.odd_with_top_bits(1024, 0x5EEDC005, synth.TAG_CAND, i) for i in range(384)]
    ns[7] = (1 << 1279) - 1 if False else ns[7]
    bases = [synth.mr_bases(n, 5, 0x5EEDC005, i) for i, n in enumerate(ns)]
    check(torch_cuda, mr, orc, ns, bases)


def test_known_primes_and_products(torch_cuda, mr, orc):
    import sympy
    ps = [sympy.nextprime(synth.odd_with_top_bits(1024, 9, synth.TAG_CAND, i)) for i in range(20)]
    m521, m607 = (1 << 521) - 1, (1 << 607) - 1
    ns = ps + [ps[0] * ps[1] % (1 << 1024) | 1, m521, m607]
    ns = [n if n.bit_length() <= 1024 else n >> (n.bit_length() - 1024) | 1 for n in ns]
    bases = [synth.mr_bases(n, 8, 10, i) for i, n in enumerate(ns)]
    v, w = check(torch_cuda, mr, orc, ns, bases)
    assert v[:20] == [1] * 20


def test_factor_verdict_and_input_rules(torch_cuda, mr, orc):
    fp = orc.base_primes(66)
    n_factor = fp[5] * ((1 << 900) + 0x1234567) | 1
    while n_factor % fp[5]:
        n_factor += 2 * fp[5]
    ns = [n_factor, 1000001, 3, (1 << 1000) + 1]          # FACTOR, even-after-fix-up-check, n < 5, odd composite
    ns[1] = 1000000                                         # even
    bases = [[2, 3], [2, 3], [2, 2], [2, (1 << 1000)]]      # last: base > n - 2
    limbs = 32
    v, w, s, _ = gpu_mr(torch_cuda, mr, ns, bases, limbs=limbs)
    assert v[0] == mr.MR_FACTOR and s[0] == 0
    assert s[1] == 5 and s[2] == 5 and s[3] == 5
    ov, _ = orc.miller_rabin(n_factor, [2, 3], orc.base_primes(66))
    assert ov == 2


def test_chernick_carmichael_1024(torch_cuda, mr, orc):
    import sympy
    t = 1 << 300
    while not (sympy.isprime(6 * t + 1) and sympy.isprime(12 * t + 1) and sympy.isprime(18 * t + 1)):
        t += 1
    n = (6 * t + 1) * (12 * t + 1) * (18 * t + 1)
    v, w = check(torch_cuda, mr, orc, [n], [synth.mr_bases(n, 6, 1, 0)])
    assert v == [0]


def test_forced_equals_compacted_early_exit(torch_cuda, mr):
    """the early-exit path (round 0 for all, then compacted (survivor, round) items) and the forced path
    (every round in one tile-job) give identical verdicts and witness rounds; batch spans several
    persistent CTAs with more items than window-table slots."""
    import ctypes
    import sympy
    torch = torch_cuda
    ns = [synth.odd_with_top_bits(512, 21, synth.TAG_CAND, i) for i in range(1500)]
    ns[::5] = [sympy.nextprime(n) for n in ns[::5]]                    # 300 planted primes
    rounds = 12
    limbs = 16
    bases = np.stack([mr.ints_to_limbs(synth.mr_bases(n, rounds, 22, i), limbs) for i, n in enumerate(ns)])
    d_n = torch.from_numpy(mr.ints_to_limbs(ns, limbs).view(np.int32)).cuda()
    d_b = torch.from_numpy(np.ascontiguousarray(bases).view(np.int32)).cuda()
    L = mr.lib()
    L.mr_internal_miller_rabin.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    out = {}
    for forced in (0, 1):
        v = torch.full((len(ns),), 9, dtype=torch.uint8, device="cuda")
        w = torch.full((len(ns),), 99, dtype=torch.int16, device="cuda")
        rc = L.mr_internal_miller_rabin(d_n.data_ptr(), limbs, len(ns), d_b.data_ptr(), rounds, 0, v.data_ptr(),
                                        w.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream, forced, 4)
        assert rc == 0
        torch.cuda.synchronize()
        out[forced] = (v.cpu().numpy().tolist(), w.cpu().numpy().tolist())
    assert out[0] == out[1]
    assert out[0][0] == [1 if sympy.isprime(n) else 0 for n in ns]      # 300 planted + the natural primes
    assert all(x == -1 for x, y in zip(out[0][1], out[0][0]) if y == 1)


def test_small_candidate_equal_to_base_prime(torch_cuda, mr, orc):
    """reading R14: a one-limb candidate that IS one of the RNS base primes has no n^-1 mod m_i; the library reports
    status MR_ERR_NOT_COPRIME with verdict PROBABLY_PRIME (it is a prime).  Other one-limb primes and composites in
    the same batch are decided normally (verdicts vs the oracle)."""
    k = k_for(mr, 1)
    fp = orc.base_primes(2 * k)
    import sympy
    other_p = sympy.prevprime(fp[-1] - 1000)                  # a prime below the base, not in it
    ns = [fp[0], fp[k], fp[2 * k - 1], other_p, 65521 * 65519]   # three base primes, a prime, a semiprime < 2^32
    bases = [[2, 3, 5]] * len(ns)
    v, w, s, limbs = gpu_mr(torch_cuda, mr, ns, bases, limbs=1)
    assert s[:3] == [mr.MR_ERR_NOT_COPRIME] * 3 and v[:3] == [mr.MR_PROBABLY_PRIME] * 3
    assert s[3] == 0 and v[3] == mr.MR_PROBABLY_PRIME
    ov, _ = orc.miller_rabin(ns[4], [2, 3, 5], fp)
    assert s[4] == 0 and v[4] == ov


@pytest.mark.parametrize("bits, k, primes", [(4423, 257, [4253, 4423]), (11213, 505, [9689, 11213])])
def test_wide_candidates_vs_oracle(torch_cuda, mr, orc, bits, k, primes):
    """Miller-Rabin above 4,096 bits (k = 257 / 505, channels-on-threads kernels with a per-candidate setup,
    DESIGN.md §4l; keys up to 16,128 bits): Mersenne primes 2^p - 1 (known primes: every round passes), random
    odd composites, a FACTOR candidate (divisible by a base prime, reading R14) and a candidate with a base outside
    [2, n-2] (status MR_ERR_RANGE); verdict and first witnessing round vs the oracle with the same explicit bases.
    20 candidates = two 16-candidate CTAs (the second ragged)."""
    import random
    rng = random.Random(bits)
    L = (bits + 31) // 32
    fp = orc.base_primes(2 * k)
    ns = [(1 << e) - 1 for e in primes]
    while len(ns) < 17:
        ns.append(rng.getrandbits(bits) | (1 << (bits - 1)) | 1)
    nf = fp[3] * (rng.getrandbits(bits - 40) | (1 << (bits - 41)) | 1)
    ns.append(nf)                                                   # FACTOR
    ns.append(rng.getrandbits(bits) | (1 << (bits - 1)) | 1)        # bad base below
    ns.append((1 << primes[0]) - 1)
    R = 3
    bases = [[rng.randrange(2, n - 1) for _ in range(R)] for n in ns]
    bases[18][1] = 1                                                # outside [2, n-2]
    v, w, s, limbs = gpu_mr(torch_cuda, mr, ns, bases, limbs=L)
    assert v[0] == v[1] == v[19] == mr.MR_PROBABLY_PRIME and w[0] == w[1] == -1
    assert v[17] == mr.MR_FACTOR and s[18] == mr.MR_ERR_RANGE and v[18] == mr.MR_COMPOSITE
    for i in list(range(17)) + [17, 19]:
        ov, ow = orc.miller_rabin(ns[i], bases[i], fp)
        assert (v[i], w[i]) == (ov, ow), i
        assert s[i] == 0
