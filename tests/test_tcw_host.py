"""CPU pins of the tensor-core wide kernel's host images (mr_tcw.cuh; k = 97, 129, 257 and 505).

Each image is the byte-split B operand of one contraction (mr_internal.h tcw_*): row (output o, byte b), K byte
(input word i, byte a) = byte b of 2^(8a) A(i, o) mod m_o.  The test decodes the exported image with an
independent python mirror of the documented slab layout, runs the u8 x u8 -> integer contraction the tensor core
performs (numpy, exact int64) on random input words, recombines the four byte columns and checks the result
against the DEFINITION of each contraction written with CPython integers from the base primes:

  BE1   Σ_i x_i |M_i|_{m'_j} |N M^-1 λ_j| 2^32 ≡ V_j (mod m'_j);  column k: Σ_i x_i |M_i|_{2^32} ≡ V_k (mod 2^32)
  BE2   (Σ_j x_j |M'_j|_{m_i} + x_k (m_i - |M'|_{m_i})) 2^32 ≡ V_i (mod m_i)
  TRN   Σ_l x_l 2^(32 l) 2^32 (× λ_c on B') ≡ V_c (mod m_c)
  EXT   Σ_p D[p] 2^(8p) ≡ Σ_j x_j M'_j + x_k (2^(32(k+1)) - M')  (mod 2^(32(k+1)))

plus the accumulator bound the kernel's epilogues rely on (every D value < 2^31).  No GPU needed.
"""
import ctypes
import random

import numpy as np
import pytest

from test_abi_host import _layout, _lib, _tables

BE1, BE2, TRN, EXT = 0, 1, 2, 3


# ---- python mirror of the mr_internal.h tcw_* geometry (the contract between the host images and the kernel)
def kp(k):
    return (4 * k + 4 + 31) & ~31


def ksteps(k):
    return kp(k) // 32


def nslab(k):
    return (ksteps(k) + 3) // 4


def steps(k, s):
    return 4 if s + 1 < nslab(k) else ksteps(k) - 4 * s


def bsw(k):
    return (k + 3) & ~3 if k <= 257 else 0   # k = 505: B residues in a global scratch slot, not in TMEM


def nout(k, e):
    return {BE1: k + 1, BE2: k, TRN: 2 * k, EXT: k + 1}[e]


def tiles(k):
    return 1 if k > 129 else 2


def ocmax(k):
    return min((((512 // tiles(k) - bsw(k)) & ~15) // 4) & ~3, 64)


def nchunks(k, e):
    return -(-nout(k, e) // ocmax(k))


def oc(k, e):
    return (-(-nout(k, e) // nchunks(k, e)) + 3) & ~3


def outn(k, e, c):
    return min(oc(k, e), nout(k, e) - c * oc(k, e))


def nc(k, e, c):
    return (4 * outn(k, e, c) + 15) & ~15


def blk_off(k, e, c, s):
    o = sum(nc(k, e, cc) * kp(k) for cc in range(c))
    return o + sum(nc(k, e, c) * 32 * steps(k, ss) for ss in range(s))


def dense(k, e, img):
    """the image as a [4 nout][kp] byte matrix (row 4 o + b), decoded from the slab blocks"""
    out = np.zeros((4 * nout(k, e), kp(k)), dtype=np.int64)
    for c in range(nchunks(k, e)):
        for s in range(nslab(k)):
            st = steps(k, s)
            blk = img[blk_off(k, e, c, s): blk_off(k, e, c, s) + nc(k, e, c) * 32 * st]
            # (r / 8) SBO + (kl / 16) 128 + (r % 8) 16 + kl % 16 with SBO = steps 256
            b = blk.reshape(nc(k, e, c) // 8, 2 * st, 8, 16).transpose(0, 2, 1, 3).reshape(nc(k, e, c), 32 * st)
            rows = 4 * outn(k, e, c)
            out[4 * c * oc(k, e): 4 * c * oc(k, e) + rows, 128 * s: 128 * s + 32 * st] = b[:rows]
            assert not b[rows:].any(), "padding rows of a chunk must be zero"
    return out


def image(k, e, N=None, limbs=0):
    mr, L = _lib()
    L.mr_internal_tcw_image.restype = ctypes.c_int
    P8 = ctypes.POINTER(ctypes.c_uint8)
    P32 = ctypes.POINTER(ctypes.c_uint32)
    nl = None
    if N is not None:
        nl = np.frombuffer(N.to_bytes(4 * limbs, "little"), dtype=np.uint32).copy()
    arg = nl.ctypes.data_as(P32) if nl is not None else None
    n = L.mr_internal_tcw_image(k, e, arg, limbs, None, 0)
    assert n > 0, n
    img = np.zeros(n, dtype=np.uint8)
    assert L.mr_internal_tcw_image(k, e, arg, limbs, img.ctypes.data_as(P8), n) == n
    assert n == blk_off(k, e, nchunks(k, e), 0)
    return img


def contract(k, e, img, xs):
    """D = bytes(x) · image^T, the u8 x u8 -> s32 products the tensor core sums (exact in int64)"""
    A = np.zeros((len(xs), kp(k)), dtype=np.int64)
    for r, x in enumerate(xs):
        for w, v in enumerate(x):
            for a in range(4):
                A[r, 4 * w + a] = (v >> (8 * a)) & 0xFF
    D = A @ dense(k, e, img).T
    assert D.max() < 2 ** 31
    return D


def combine(D, o):
    return sum(int(D[4 * o + b]) << (8 * b) for b in range(4))


@pytest.fixture(scope="module", params=[97, 129, 257, 505])
def base(request):
    k = request.param
    flat, primes, _ = _tables(k)
    B, Bp = primes[:k], primes[k:]
    M, Mp = 1, 1
    for m in B:
        M *= m
    for m in Bp:
        Mp *= m
    return k, B, Bp, M, Mp


def test_geometry_fits(base):
    k = base[0]
    assert tiles(k) * (max(nc(k, e, c) for e in range(4) for c in range(nchunks(k, e))) + bsw(k)) <= 512
    assert kp(k) >= 4 * k + 4 and all(oc(k, e) % 4 == 0 for e in range(4))


def test_be1_image_definition(base):
    k, B, Bp, M, Mp = base
    rng = random.Random(k)
    bits = 32 * (k - 1) - 40
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    limbs = (bits + 31) // 32
    img = image(k, BE1, N, limbs)
    xs = [[rng.getrandbits(32) for _ in range(k)] + [rng.getrandbits(32)] for _ in range(3)]   # word k: ignored
    D = contract(k, BE1, img, xs)
    W = 1 << 32
    for r, x in enumerate(xs):
        for j in [0, 1, k - 2, k - 1] + rng.sample(range(k), 6):
            m = Bp[j]
            lam = pow(Mp // m, -1, m)
            nu = N * pow(M, -1, m) * lam % m                       # |N M^-1 λ_j|
            want = sum(x[i] * ((M // B[i]) % m) for i in range(k)) * nu * W % m
            assert combine(D[r], j) % m == want
        assert combine(D[r], k) % W == sum(x[i] * ((M // B[i]) % W) for i in range(k)) % W


def test_be1_epilogue_sum_fits_64_bits(base):
    """the BE1 epilogue forms t*_j (C1_j 2^64 mod m'_j) + V_j in ONE 64-bit multiply-add (mr_tcw.cuh, mad.wide.u32): t* is
    a lazy residue < 2^32 and V = Σ_b 2^(8b) D_b with every D_b <= 4k 255^2 (4k u8 x u8 products per column), so the sum
    fits only because every per-k constant C1_j 2^64 mod m'_j stays far enough below 2^32 — pinned here from the base
    table (reading R1's primes), at every tensor-wide k"""
    k, B, Bp, M, Mp = base
    flat, primes, _ = _tables(k)
    o_c1 = _layout(k)["C1"]
    vmax = 4 * k * 255 * 255 * (1 + 2 ** 8 + 2 ** 16 + 2 ** 24)
    for j in range(k):
        m = Bp[j]
        c1 = int(flat[o_c1 + j])
        assert c1 == pow(M, -1, m) * pow(pow(Mp // m, -1, m), -1, m) % m   # C1_j = |M^-1 λ_j^-1|_{m'_j}
        xw = c1 * pow(2, 64, m) % m
        assert (2 ** 32 - 1) * xw + vmax < 2 ** 64, (k, j)


def test_be2_image_definition(base):
    k, B, Bp, M, Mp = base
    rng = random.Random(k + 1)
    img = image(k, BE2)
    xs = [[rng.getrandbits(32) for _ in range(k)] + [rng.randrange(k + 1)] for _ in range(3)]  # word k = α' <= k
    D = contract(k, BE2, img, xs)
    W = 1 << 32
    for r, x in enumerate(xs):
        for i in [0, 1, k - 1] + rng.sample(range(k), 6):
            m = B[i]
            want = (sum(x[j] * ((Mp // Bp[j]) % m) for j in range(k)) + x[k] * ((m - Mp % m) % m)) * W % m
            assert combine(D[r], i) % m == want


def test_trn_image_definition(base):
    k, B, Bp, M, Mp = base
    rng = random.Random(k + 2)
    img = image(k, TRN)
    xs = [[rng.getrandbits(32) for _ in range(k - 1)] + [0, 0] for _ in range(3)]   # an input of k - 1 limbs
    D = contract(k, TRN, img, xs)
    W = 1 << 32
    for r, x in enumerate(xs):
        X = sum(v << (32 * l) for l, v in enumerate(x[:k]))
        for c in [0, k - 1, k, 2 * k - 1] + rng.sample(range(2 * k), 6):
            m = (B + Bp)[c]
            want = X * W % m
            if c >= k:
                want = want * pow(Mp // m, -1, m) % m                   # ξ-form of the B' residues
            assert combine(D[r], c) % m == want


def test_ext_image_definition(base):
    k, B, Bp, M, Mp = base
    rng = random.Random(k + 3)
    img = image(k, EXT)
    xs = [[rng.getrandbits(32) for _ in range(k)] + [rng.randrange(k + 1)] for _ in range(3)]
    D = contract(k, EXT, img, xs)
    R = 1 << (32 * (k + 1))
    for r, x in enumerate(xs):
        X = sum(int(D[r][p]) << (8 * p) for p in range(4 * (k + 1))) % R
        want = (sum(x[j] * (Mp // Bp[j]) for j in range(k)) + x[k] * (R - Mp)) % R
        assert X == want


def test_image_errors():
    mr, L = _lib()
    L.mr_internal_tcw_image.restype = ctypes.c_int
    assert L.mr_internal_tcw_image(65, 1, None, 0, None, 0) < 0       # not a tensor-wide k
    assert L.mr_internal_tcw_image(97, 4, None, 0, None, 0) < 0       # no such extension
    assert L.mr_internal_tcw_image(97, 0, None, 0, None, 0) < 0       # BE1 needs a modulus
