"""CPU-side checks of the boundary: the shared library loads, exports every symbol declared in
include/mr_rns.h, reports errors without a GPU, and its host-side precomputation satisfies the
identities of DESIGN.md §3 (checked with independent CPython arithmetic, no oracle involvement
needed: these are definitions of the tables, not results of the method)."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

from conftest import ROOT

HDR = os.path.join(ROOT, "include", "mr_rns.h")


def _lib():
    import paper_1305_3699_b200 as mr
    return mr, mr.lib()


def test_exports_every_header_symbol():
    mr, L = _lib()
    src = open(HDR).read()
    names = set(re.findall(r"\b(mr_[a-z0-9_]+)\s*\(", src))
    assert {"mr_rns_ctx_create", "mr_modexp_batch", "mr_rsa_encrypt_batch", "mr_rsa_decrypt_batch",
            "mr_miller_rabin_batch"} <= names
    for n in names:
        assert hasattr(L, n), n
    assert set(mr.EXPORTS) == names


def test_strerror_and_supported_k():
    mr, L = _lib()
    assert mr.mr_strerror(0) == "ok"
    assert "range" in mr.mr_strerror(5)
    ks = mr.mr_rns_supported_k()
    assert ks == sorted(ks) and 33 in ks and 65 in ks


def test_no_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mr, L = _lib()
    with pytest.raises(mr.MrError) as e:
        mr.mr_rns_ctx_create(3233, 1)
    assert e.value.code == mr.MR_ERR_CUDA
    with pytest.raises(mr.MrError) as e:
        mr.mr_rns_ctx_create(3232, 1)                  # even modulus is rejected before any device work
    assert e.value.code == mr.MR_ERR_EVEN_MODULUS


def test_argument_errors():
    mr, L = _lib()
    h = ctypes.c_void_p()
    assert L.mr_rns_ctx_create(ctypes.byref(h), None, 1, 0, 0) == mr.MR_ERR_ARG
    assert L.mr_modexp_batch(None, None, None, 0, None, 0, None, None) == mr.MR_ERR_ARG
    assert L.mr_rsa_decrypt_batch(None, None, None, 0, None, None) == mr.MR_ERR_ARG


def _tables(k):
    mr, L = _lib()
    L.mr_internal_base_table.restype = ctypes.c_int
    L.mr_internal_ctx_table.restype = ctypes.c_int
    n = L.mr_internal_base_table(k, None, 0, None)
    flat = np.zeros(n, dtype=np.uint32)
    primes = np.zeros(2 * k, dtype=np.uint32)
    P = ctypes.POINTER(ctypes.c_uint32)
    L.mr_internal_base_table(k, flat.ctypes.data_as(P), n, primes.ctypes.data_as(P))
    npow = L.mr_internal_pow_table(k, None, 0)
    pw = np.zeros(npow, dtype=np.uint32)
    L.mr_internal_pow_table(k, pw.ctypes.data_as(P), npow)
    return flat, [int(p) for p in primes], pw


def _layout(k):
    """python mirror of mr_internal.h base_layout (prefix = __constant__ bank)."""
    o = {}
    o["c"] = 0
    o["c2"] = 2 * k
    o["A1r"] = 4 * k
    o["A2r"] = o["A1r"] + k
    o["C1"] = o["A2r"] + k
    o["pin"] = o["C1"] + k
    o["misc"] = o["pin"] + k
    o["NMp"] = o["misc"] + 4
    o["MiS"] = o["NMp"] + k + 1
    o["MU"] = o["MiS"] + k
    o["ONE"] = o["MU"] + k
    o["ML"] = o["ONE"] + 2 * k + 1
    o["MM"] = o["ML"] + k + 1
    o["MINV"] = o["MM"] + 2 * k
    o["XW"] = o["MINV"] + 2 * k
    o["A2C"] = o["XW"] + k
    o["MpL"] = o["A2C"] + k
    o["A1"] = o["MpL"] + k * (k + 1)
    o["A2"] = o["A1"] + k * k
    return o


@pytest.mark.parametrize("k", [1, 3, 17, 33, 97])
def test_base_table_identities(k):
    import sympy
    flat, primes, pw = _tables(k)
    B, Bp = primes[:k], primes[k:]
    # reading R1: the 2k largest primes below 2^32 (= 3 mod 4 only, for k <= 65), descending
    expect, x = [], 1 << 32
    while len(expect) < 2 * k:
        x = sympy.prevprime(x)
        if k > 65 or x % 4 == 3:
            expect.append(x)
    assert primes == expect
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    o = _layout(k)
    f = [int(v) for v in flat]
    W = 1 << 32
    for ch, m in enumerate(B + Bp):
        assert f[o["c"] + ch] == W - m and f[o["c2"] + ch] == (W - m) ** 2
        assert f[o["MM"] + ch] == m and f[o["MINV"] + ch] * m % W == W - 1     # -m^-1 mod 2^32
    for i in range(k):
        Mi = M // B[i]
        for j in range(k):
            assert f[o["A1"] + i * k + j] == Mi % Bp[j]
        assert f[o["A1r"] + i] == Mi % W
    for j in range(k):
        Mpj = Mp // Bp[j]
        for i in range(k):
            assert f[o["A2"] + j * k + i] == Mpj % B[i]
        assert f[o["A2r"] + j] == Mpj % W
        lam = pow(Mpj, -1, Bp[j])
        assert f[o["C1"] + j] == pow(M, -1, Bp[j]) * pow(lam, -1, Bp[j]) % Bp[j]
        assert f[o["XW"] + j] == f[o["C1"] + j] * (W * W % Bp[j]) % Bp[j]
        limbs = sum(f[o["MpL"] + j * (k + 1) + l] << (32 * l) for l in range(k + 1))
        assert limbs == Mpj
    for i in range(k):
        assert (f[o["pin"] + i] + Mp) % B[i] == 0                      # m_i - |M'|_{m_i}
    assert f[o["misc"]] * M % W == 1 and f[o["misc"] + 1] * Mp % W == 1
    nmp = sum(f[o["NMp"] + l] << (32 * l) for l in range(k + 1))
    assert nmp + Mp == 1 << (32 * (k + 1))
    assert sum(f[o["ML"] + l] << (32 * l) for l in range(k + 1)) == M
    for i in range(k):
        assert f[o["MiS"] + i] == (M // B[i]) % B[i] and f[o["ONE"] + i] == 1
    for j in range(k):
        assert f[o["MU"] + j] == pow(M, -1, Bp[j])
        assert f[o["ONE"] + k + j] == pow(Mp // Bp[j], -1, Bp[j])
    assert f[o["ONE"] + 2 * k] == 1
    # to_rns powers: |2^(32 l)|_{m_i} and |2^(32 l) λ_j|_{m'_j}
    for l in range(k):
        for i in range(k):
            assert int(pw[l * 2 * k + i]) == pow(2, 32 * l, B[i])
        for j in range(k):
            lam = pow(Mp // Bp[j], -1, Bp[j])
            assert int(pw[l * 2 * k + k + j]) == pow(2, 32 * l, Bp[j]) * lam % Bp[j]
    # capacity headroom of reading R5: 4 (k+3)^2 N < M leaves ~20 bits for N of 32(k-1) bits
    if k >= 17:
        assert 4 * (k + 3) ** 2 * (1 << (32 * (k - 1))) < M


@pytest.mark.parametrize("name", ["rsa1024", "rsa2048"])
def test_ctx_table_identities(keys, name):
    mr, L = _lib()
    key = keys[name]
    N = key["n"] if name == "rsa1024" else key["p"]          # 1024-bit moduli -> k = 33
    k = 33
    flat, primes, _ = _tables(k)
    B, Bp = primes[:k], primes[k:]
    limbs = (N.bit_length() + 31) // 32
    P = ctypes.POINTER(ctypes.c_uint32)
    nl = np.frombuffer(N.to_bytes(4 * limbs, "little"), dtype=np.uint32).copy()
    nw = L.mr_internal_ctx_table(nl.ctypes.data_as(P), limbs, k, None, 0)
    assert nw > 0
    cx = np.zeros(nw, dtype=np.uint32)
    L.mr_internal_ctx_table(nl.ctypes.data_as(P), limbs, k, cx.ctypes.data_as(P), nw)
    cx = [int(v) for v in cx]
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    W = 1 << 32
    assert cx[0] == k and cx[1] == limbs
    assert cx[4] == N * pow(M, -1, W) % W
    sig, c2, r2, one = 8, 8 + k, 8 + 2 * k, 8 + 2 * k + 2 * k + 1
    for i in range(k):
        assert cx[sig + i] * N * (M // B[i]) % B[i] == B[i] - 1       # σ_i N M_i = -1 (mod m_i)
    for j in range(k):
        lam = pow(Mp // Bp[j], -1, Bp[j])
        assert cx[c2 + j] == N * pow(M, -1, Bp[j]) * lam % Bp[j]
    R2 = M * M % N
    for i in range(k):
        assert cx[r2 + i] == R2 % B[i] and cx[one + i] == 1
    for j in range(k):
        lam = pow(Mp // Bp[j], -1, Bp[j])
        assert cx[r2 + k + j] == R2 % Bp[j] * lam % Bp[j] and cx[one + k + j] == lam
    assert cx[r2 + 2 * k] == R2 % W
    _check_tensor_constants(cx, k, N, B, Bp, M, Mp, sig, r2, one)


def _cx_tc_offsets(k):
    """python mirror of the tensor-path part of mr_internal.h cx_* (DESIGN.md §4e, §4g)."""
    inb = 8 + 2 * k + 4 * (2 * k + 1) + k + 1
    sc = inb + 2 * k + 2
    a1x = (sc + 4 * (2 * k + 1) + 1) & ~1
    a2s = a1x + 2 * k
    scv = a2s + k
    ep1 = (scv + 4 + 3) & ~3
    ep2 = ep1 + 4 * k
    return {"sc": sc, "a1x": a1x, "a2s": a2s, "scv": scv, "ep1": ep1, "ep2": ep2}


def _check_tensor_constants(cx, k, N, B, Bp, M, Mp, sig, r2, one):
    """ρ-scaling with word-Montgomery factors: ρ_i² = ε_i σ_i 2^32 (mod m_i); the scaled constant
    vectors; the signed m_r column; the epilogue constants (m, -m^-1 mod 2^32, C1 2^64, |M'_j|_{2^32})."""
    W = 1 << 32
    o = _cx_tc_offsets(k)
    n = 2 * k + 1
    for i, m in enumerate(B):
        rho = cx[o["sc"] + 1 * n + i]                                  # ONE scaled once: ρ_i
        v = rho * rho % m
        eps = 1 if v == cx[sig + i] * W % m else -1
        assert v == eps * cx[sig + i] * W % m                          # ρ² = ε σ 2^32
        assert m % 4 == 3                                              # reading R1 (k <= 65)
        assert cx[o["sc"] + 0 * n + i] == cx[r2 + i] * v % m           # R² ρ² (operand right after to_rns)
        assert cx[o["sc"] + 3 * n + i] == cx[r2 + i] * rho % m         # R² ρ (loaded accumulator)
        assert cx[o["a1x"] + 2 * i] == (eps * ((M // m) % W)) % W       # ε_i |M_i|_{2^32}
    for ch in range(n):                                                # B' and m_r channels unscaled
        if ch >= k:
            assert cx[o["sc"] + 0 * n + ch] == cx[r2 + ch] and cx[o["sc"] + 1 * n + ch] == cx[one + ch]
    for j, m in enumerate(Bp):
        lam = pow(Mp // m, -1, m)
        c1 = pow(M, -1, m) * pow(lam, -1, m) % m
        e = cx[o["ep1"] + 4 * j: o["ep1"] + 4 * j + 4]
        assert e[0] == m and e[1] * m % W == W - 1 and e[2] == c1 * W * W % m and e[3] == (Mp // m) % W
    for i, m in enumerate(B):
        assert cx[o["ep2"] + 2 * i] == m and cx[o["ep2"] + 2 * i + 1] * m % W == W - 1


def test_ctx_table_rejections():
    mr, L = _lib()
    P = ctypes.POINTER(ctypes.c_uint32)
    _, primes, _ = _tables(33)
    bad = primes[5] * ((1 << 900) + 1)                          # shares a base prime
    while bad % 2 == 0:
        bad += primes[5]
    limbs = (bad.bit_length() + 31) // 32
    nl = np.frombuffer(bad.to_bytes(4 * limbs, "little"), dtype=np.uint32).copy()
    assert L.mr_internal_ctx_table(nl.ctypes.data_as(P), limbs, 33, None, 0) == -mr.MR_ERR_NOT_COPRIME
    big = (1 << 1100) + 1
    limbs = 35
    nl = np.frombuffer(big.to_bytes(4 * limbs, "little"), dtype=np.uint32).copy()
    assert L.mr_internal_ctx_table(nl.ctypes.data_as(P), limbs, 33, None, 0) == -mr.MR_ERR_CAPACITY


def _wide_layout(k):
    """python mirror of mr_internal.h wide_layout."""
    o = {"mm": 0}
    o["minv"] = o["mm"] + 2 * k
    o["r32"] = o["minv"] + 2 * k
    o["xw"] = o["r32"] + 2 * k
    o["a1r"] = o["xw"] + k
    o["a2r"] = o["a1r"] + k
    o["pinw"] = o["a2r"] + k
    o["misc"] = o["pinw"] + k
    o["a2w"] = (o["misc"] + 4 + 3) & ~3
    o["pow"] = o["a2w"] + _wch_rows(k) * k
    o["mpl"] = o["pow"] + _wch_rows(k) * 2 * k
    o["nmp"] = o["mpl"] + _wch_rows(k) * (k + 1)
    o["a1w"] = (o["nmp"] + k + 1 + 3) & ~3
    o["lam"] = o["a1w"] + _wch_rows(k) * k
    o["mu"] = o["lam"] + k
    o["mis"] = o["mu"] + k
    o["ml"] = o["mis"] + k
    o["one"] = o["ml"] + k + 1
    o["words"] = o["one"] + 2 * k + 1
    return o


def _wch_rows(r):
    return (r + 7) & ~7


def _wch_at(i, j, ncols):
    """mr_internal.h wch_at: chunked [R][C] matrix, rows in groups of 8, element (i, j) at
    ((i // 8) C + j) 8 + i % 8."""
    return ((i >> 3) * ncols + j) * 8 + (i & 7)


def test_wide_table_identities():
    """host constants of the wide-operand kernel (k = 257): word-Montgomery constants
    with their 2^32 factors folded in, checked against the definitions on sampled entries."""
    mr, L = _lib()
    k = 257
    assert 257 in mr.mr_rns_supported_k() and 505 in mr.mr_rns_supported_k()
    P = ctypes.POINTER(ctypes.c_uint32)
    L.mr_internal_wide_table.restype = ctypes.c_int
    n = L.mr_internal_wide_table(k, None, 0)
    o = _wide_layout(k)
    assert n == o["words"]
    t = np.zeros(n, dtype=np.uint32)
    L.mr_internal_wide_table(k, t.ctypes.data_as(P), n)
    t = [int(v) for v in t]
    _, primes, _ = _tables(k)
    B, Bp = primes[:k], primes[k:]
    W = 1 << 32
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    rng = np.random.default_rng(257)
    for ch in list(range(4)) + [int(v) for v in rng.integers(0, 2 * k, 20)]:
        m = (B + Bp)[ch]
        assert t[o["mm"] + ch] == m and t[o["minv"] + ch] * m % W == W - 1 and t[o["r32"] + ch] == W % m
    for j in [0, 1, k - 1] + [int(v) for v in rng.integers(0, k, 8)]:
        m = Bp[j]
        lam = pow(Mp // m, -1, m)
        c1 = pow(M, -1, m) * pow(lam, -1, m) % m
        assert t[o["xw"] + j] == c1 * W * W % m and t[o["a2r"] + j] == (Mp // m) % W
        for i in [0, k - 1] + [int(v) for v in rng.integers(0, k, 4)]:
            assert t[o["a2w"] + _wch_at(j, i, k)] == (Mp // m) % B[i] * W % B[i]
    for i in [0, k - 1]:
        assert t[o["pinw"] + i] == (B[i] - Mp % B[i]) % B[i] * W % B[i] and t[o["a1r"] + i] == (M // B[i]) % W
    for l in [0, 1, k - 1]:
        for ch in [0, k - 1, k, 2 * k - 1]:
            m = (B + Bp)[ch]
            v = pow(2, 32 * (l + 1), m)
            if ch >= k:
                v = v * pow(Mp // m, -1, m) % m
            assert t[o["pow"] + _wch_at(l, ch, 2 * k)] == v
    assert sum(t[o["nmp"] + l] << (32 * l) for l in range(k + 1)) + Mp == 1 << (32 * (k + 1))
    for j in [0, k - 1] + [int(v) for v in rng.integers(0, k, 4)]:   # M'_j positional limbs
        m = Bp[j]
        assert sum(t[o["mpl"] + _wch_at(j, l, k + 1)] << (32 * l) for l in range(k + 1)) == Mp // m
    # Miller-Rabin section: unmerged BE1 A1_ij 2^32 mod m'_j, λ_j, μ_j, |M_i|_{m_i}, M limbs, the image of 1
    for j in [0, k - 1] + [int(v) for v in rng.integers(0, k, 3)]:
        m = Bp[j]
        assert t[o["lam"] + j] == pow(Mp // m, -1, m) and t[o["mu"] + j] == pow(M, -1, m)
        for i in [0, k - 1] + [int(v) for v in rng.integers(0, k, 3)]:
            assert t[o["a1w"] + _wch_at(i, j, k)] == (M // B[i]) % m * W % m
    for i in [0, k - 1]:
        assert t[o["mis"] + i] == (M // B[i]) % B[i]
    assert sum(t[o["ml"] + l] << (32 * l) for l in range(k + 1)) == M
    assert [t[o["one"] + c] for c in (0, k - 1, 2 * k)] == [1, 1, 1]
    assert t[o["one"] + k] == pow(Mp // Bp[0], -1, Bp[0])
    pad = [t[o["a2w"] + _wch_at(i, j, k)] for i in range(k, _wch_rows(k)) for j in (0, k - 1)]
    assert not any(pad)                                                # zero rows up to the group size
    assert L.mr_internal_wide_table(65, None, 0) < 0 and L.mr_internal_wide_table(129, None, 0) > 0


def test_keygen_drbg_argument_errors():
    mr, L = _lib()
    assert L.mr_rsa_keygen_batch_drbg(None, 1, 1024, 65537, 5, *([None] * 7), 0, None) == mr.MR_ERR_ARG


class _FakeCuda:
    """Just enough of a torch CUDA tensor for the binding's argument checks (no device needed)."""

    def __init__(self, shape, itemsize=4, device=0):
        import math
        self.shape, self.is_cuda, self._n = tuple(shape), True, math.prod(shape)
        self.dtype = type("dt", (), {"itemsize": itemsize})()
        self.device = type("dev", (), {"index": device})()

    def is_contiguous(self):
        return True

    def dim(self):
        return len(self.shape)

    def numel(self):
        return self._n

    def data_ptr(self):
        return 0x1000


def test_binding_validates_device_buffers():
    """the C ABI cannot see tensor sizes, so the binding checks element size, 2-D width,
    element count and device before any pointer crosses it."""
    mr, _ = _lib()
    ok = _FakeCuda((10, 32))
    assert mr._arg(ok, "x", 4, 10 * 32, 32, 0) == 0x1000
    assert mr._arg(None, "x", 4, 1) is None
    for bad, why in ((_FakeCuda((10, 32), itemsize=8), "8-byte"), (_FakeCuda((320,)), "1-D"),
                     (_FakeCuda((10, 31)), "width"), (_FakeCuda((9, 32)), "short"),
                     (_FakeCuda((10, 32), device=1), "device")):
        with pytest.raises(mr.MrError) as e:
            mr._arg(bad, "x", 4, 10 * 32, 32, 0)
        assert e.value.code == mr.MR_ERR_ARG, why
    with pytest.raises(mr.MrError):
        mr.mr_modexp_batch(ctypes.c_void_p(12345), ok, ok, 10, 3)        # handle not created here


@pytest.mark.parametrize("k", [17, 33, 49, 65])
def test_fractional_alpha_bound(k):
    """reading R2b: the tensor kernels take α' = floor(Σ_j ξ'_j / m'_j) as (Σ_j (ξ'_j >> 8) + 2^14) >> 24.  Exact iff
    (1) the approximation error stays below the 2^-10 offset: Σ_j ξ'_j/m'_j - Σ_j (ξ'_j >> 8)/2^24 < k (max c'_j/m'_j
    + 2^-24) for lazy ξ'_j < 2^32, and (2) r/M' + 2^-10 < 1 for every value r < (2k+3)N that is extended, with N the
    largest modulus ctx_create admits ((k+2)^2 N < M, (k+2) N < M').  Checked from the base primes, plus brute force of
    the formula on random residue vectors of values r near the bound (exact rational arithmetic)."""
    from fractions import Fraction
    _, primes, _ = _tables(k)
    B, Bp = primes[:k], primes[k:]
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    err = sum(Fraction((1 << 32) - m, m) + Fraction(1, 1 << 24) for m in Bp)
    assert err < Fraction(1, 1 << 10)
    nmax = min((M - 1) // (k + 2) ** 2, (Mp - 1) // (k + 2))
    assert Fraction((2 * k + 3) * nmax, Mp) + Fraction(1, 1 << 10) < 1
    rng = random.Random(k)
    for _ in range(200):
        r = rng.randrange((2 * k + 3) * nmax)
        # lazy ξ'_j: the canonical value or + m'_j when that still fits 32 bits
        xs = []
        for m in Bp:
            Mj = Mp // m
            x = r * pow(Mj, -1, m) % m
            if x + m < (1 << 32) and rng.random() < 0.5:
                x += m
            xs.append(x)
        alpha = (sum(x >> 8 for x in xs) + (1 << 14)) >> 24
        exact = sum(x * (Mp // m) for x, m in zip(xs, Bp)) - r
        assert exact % Mp == 0 and exact // Mp == alpha


@pytest.mark.parametrize("k", [97, 129, 257, 505])
def test_fractional_alpha_bound_wide(k):
    """reading R2b in the tensor-core wide kernel (mr_tcw.cuh W_FSH): α' = (Σ_j (ξ'_j >> sh) + 2^(26 - sh)) >> (32 - sh)
    with sh = 8 / 9 / 10 for k <= 129 / 257 / 505.  Exact iff the sum fits 32 bits (k < 2^sh), the approximation error
    k (max c'_j / m'_j + 2^(sh - 32)) stays below the 2^-6 offset, and r / M' + 2^-6 < 1 for the extended values r <
    (k+3) N of every admitted modulus; plus brute force on lazy residue vectors near the bound (exact arithmetic)."""
    from fractions import Fraction
    sh = 8 if k <= 129 else (9 if k <= 257 else 10)
    assert k < (1 << sh)
    _, primes, _ = _tables(k)
    B, Bp = primes[:k], primes[k:]
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    err = sum(Fraction((1 << 32) - m, m) + Fraction(1, 1 << (32 - sh)) for m in Bp)
    assert err < Fraction(1, 64)
    nmax = min((M - 1) // (k + 2) ** 2, (Mp - 1) // (k + 2))
    assert Fraction((k + 3) * nmax, Mp) + Fraction(1, 64) < 1
    rng = random.Random(k)
    for _ in range(40):
        r = rng.randrange((k + 3) * nmax)
        xs = []
        for m in Bp:
            x = r * pow(Mp // m, -1, m) % m
            if x + m < (1 << 32) and rng.random() < 0.5:
                x += m
            xs.append(x)
        s = sum(x >> sh for x in xs)
        assert s < (1 << 32)
        alpha = (s + (1 << (26 - sh))) >> (32 - sh)
        exact = sum(x * (Mp // m) for x, m in zip(xs, Bp)) - r
        assert exact % Mp == 0 and exact // Mp == alpha


@pytest.mark.parametrize("k", [17, 33, 49, 65])
def test_scaled_be1_epilogue_sum_fits_64_bits(k):
    """the ρ-scaled BE1 epilogue (mr_kernels.cuh, MR_EPI_NOFOLD) forms t*_j (C1 c'^2)_j + V_j in one 64-bit multiply-add
    with the byte-column sum V unfolded: t* < 2^32 (lazy), V <= (4k 255^2 + 128 255)(1 + 2^8 + 2^16 + 2^24) (the 4k
    digit bytes plus the offset and α' columns), so the sum fits only because every per-k constant (C1 c'^2)_j =
    C1_j 2^64 mod m'_j is far enough below 2^32 — pinned here from the base table"""
    flat, primes, _ = _tables(k)
    L = _layout(k)
    Bp = primes[k:]
    vmax = (4 * k * 255 * 255 + 128 * 255) * (1 + 2 ** 8 + 2 ** 16 + 2 ** 24)
    for j in range(k):
        m = Bp[j]
        xw = int(flat[L["XW"] + j])
        assert xw == int(flat[L["C1"] + j]) * pow(2, 64, m) % m
        assert (2 ** 32 - 1) * xw + vmax < 2 ** 64, (k, j)
