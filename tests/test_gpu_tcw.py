"""GPU parity of the tensor-core wide kernel (k_modexp_tcw, mr_tcw.cuh) for k = 97, 129, 257 and 505:
3072- / 4096- / 8192- / 16,128-bit moduli and the CRT halves of 6144- / 8192- / 16,128-bit keys.  Every case runs on the tensor path and on the
IMAD wide kernel (mr_internal_set_tcw), both compared element by element with the CPU oracle; ragged batches span
several 128-message tile-jobs, with edge inputs 0, 1, 2, N-1, N-2 and out-of-range inputs (status 5, output 0).
"""
import ctypes
import math
import os
import random
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PATHS = ["tcw", "imad_wide"]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def mr():
    import paper_1305_3699_b200 as mr
    L = mr.lib()
    L.mr_internal_set_tcw.argtypes = [ctypes.c_int]
    yield mr
    L.mr_internal_set_tcw(-1)


def set_path(mr, path):
    mr.lib().mr_internal_set_tcw(1 if path == "tcw" else 0)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def modexp(torch, mr, N, xs, E, limbs):
    ctx = mr.RnsContext(N, limbs)
    x = dev(torch, mr.ints_to_limbs(xs, limbs))
    y = torch.empty_like(x)
    st = torch.full((len(xs),), -1, dtype=torch.int32, device="cuda")
    ctx.modexp(x, y, E, d_status=st)
    torch.cuda.synchronize()
    return host(y), host(st).view(np.int32).tolist(), ctx


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("bits", [3072, 4096])
def test_tcw_modexp_vs_oracle(torch_cuda, mr, orc, bits, path):
    """ragged 389-message batch (four tile-jobs, the last with 5 messages) for E = 3, 65537 and a 400-bit E"""
    set_path(mr, path)
    rng = random.Random(bits + 11)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [0, 1, 2, N - 1, N - 2, 1 << (bits - 2)] + [rng.randrange(N) for _ in range(381)] + [N, N + 7]
    for E in (3, 65537, rng.getrandbits(400) | (1 << 399)):
        y, st, ctx = modexp(torch_cuda, mr, N, xs, E, L)
        assert ctx.k == {3072: 97, 4096: 129}[bits]
        assert st == [0] * 387 + [5, 5] and not y[387:].any()
        ref = orc.modexp_batch(mr.ints_to_limbs(xs[:387], L), E, N, threads=8)
        assert np.array_equal(y[:387], ref), (path, E.bit_length())


@pytest.mark.parametrize("path", PATHS)
def test_tcw_k257_modexp_vs_oracle(torch_cuda, mr, orc, path):
    """8192-bit modulus (k = 257: one 128-message tile per CTA, two compute warps per lane quadrant): ragged 200-message
    batch (two tile-jobs, the second with 72) with edge inputs, E = 65537 and a 160-bit E, every output vs the oracle"""
    set_path(mr, path)
    bits = 8192
    rng = random.Random(bits + 11)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [0, 1, 2, N - 1, N - 2, 1 << (bits - 2)] + [rng.randrange(N) for _ in range(192)] + [N, N + 7]
    for E in (65537, rng.getrandbits(160) | (1 << 159)):
        y, st, ctx = modexp(torch_cuda, mr, N, xs, E, L)
        assert ctx.k == 257
        assert st == [0] * 198 + [5, 5] and not y[198:].any()
        ref = orc.modexp_batch(mr.ints_to_limbs(xs[:198], L), E, N, threads=8)
        assert np.array_equal(y[:198], ref), (path, E.bit_length())


@pytest.mark.parametrize("path", PATHS)
def test_tcw_k257_crt_decrypt_vs_oracle(torch_cuda, mr, orc, path):
    """CRT decryption of a 16,128-bit key (§3.1): two 8064-bit half ladders at k = 257 in one launch, then the
    positional recombination; 140 ciphertexts with edge inputs, every output vs the oracle"""
    set_path(mr, path)
    half_bits = 8064
    rng = random.Random(half_bits + 5)
    while True:
        p = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        q = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        if p != q and math.gcd(p, q) == 1:
            break
    n, H = p * q, half_bits // 32
    dp, dq = rng.getrandbits(96) | 1, rng.getrandbits(96) | 1
    qinv = pow(q, -1, p)
    cs = [0, 1, n - 1, p, q, 2 * p, 3 * q] + [rng.randrange(n) for _ in range(132)] + [n + 1]
    key = mr.RsaPrivateKey(p, q, dp, dq, qinv)
    c = dev(torch_cuda, mr.ints_to_limbs(cs, 2 * H))
    m = torch_cuda.empty_like(c)
    st = torch_cuda.full((len(cs),), -1, dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=st)
    torch_cuda.cuda.synchronize()
    assert host(st).view(np.int32).tolist() == [0] * 139 + [5]
    ref = orc.crt_decrypt_batch(mr.ints_to_limbs(cs[:139], 2 * H), p, q, dp, dq, qinv, H, threads=8)
    got = host(m)
    assert np.array_equal(got[:139], ref) and not got[139].any()


def test_tcw_k257_paths_identical_full_exponent(torch_cuda, mr):
    """k = 257 tensor path and IMAD wide kernel give identical bytes for a full 8192-bit exponent (300 messages)"""
    rng = random.Random(257)
    N = rng.getrandbits(8192) | (1 << 8191) | 1
    xs = [rng.randrange(N) for _ in range(300)]
    E = rng.getrandbits(8192) | (1 << 8191)
    set_path(mr, "tcw")
    a, _, _ = modexp(torch_cuda, mr, N, xs, E, 256)
    set_path(mr, "imad_wide")
    b, _, _ = modexp(torch_cuda, mr, N, xs, E, 256)
    assert np.array_equal(a, b)
    for i in (0, 150, 299):
        assert int.from_bytes(a[i].tobytes(), "little") == pow(xs[i], E, N)


@pytest.mark.parametrize("path", PATHS)
def test_tcw_k505_modexp_vs_oracle(torch_cuda, mr, orc, path):
    """16,128-bit modulus (k = 505: 64-message tiles, M = 64 MMAs, B residues in the global scratch slot): ragged
    100-message batch (two tile-jobs, the second with 36) with edge inputs, E = 65537 and a 96-bit E, vs the oracle"""
    set_path(mr, path)
    bits = 16128
    rng = random.Random(bits + 11)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [0, 1, 2, N - 1, N - 2, 1 << (bits - 2)] + [rng.randrange(N) for _ in range(92)] + [N, N + 7]
    for E in (65537, rng.getrandbits(96) | (1 << 95)):
        y, st, ctx = modexp(torch_cuda, mr, N, xs, E, L)
        assert ctx.k == 505
        assert st == [0] * 98 + [5, 5] and not y[98:].any()
        ref = orc.modexp_batch(mr.ints_to_limbs(xs[:98], L), E, N, threads=8)
        assert np.array_equal(y[:98], ref), (path, E.bit_length())


def test_tcw_k505_paths_identical_full_exponent(torch_cuda, mr):
    """k = 505 tensor path and IMAD wide kernel give identical bytes for a full 16,128-bit exponent (70 messages)"""
    rng = random.Random(505)
    N = rng.getrandbits(16128) | (1 << 16127) | 1
    xs = [rng.randrange(N) for _ in range(70)]
    E = rng.getrandbits(16128) | (1 << 16127)
    set_path(mr, "tcw")
    a, _, _ = modexp(torch_cuda, mr, N, xs, E, 504)
    set_path(mr, "imad_wide")
    b, _, _ = modexp(torch_cuda, mr, N, xs, E, 504)
    assert np.array_equal(a, b)
    assert int.from_bytes(a[69].tobytes(), "little") == pow(xs[69], E, N)


@pytest.mark.parametrize("count", [1, 127, 128, 129])
def test_tcw_batch_edges(torch_cuda, mr, orc, count):
    """single-tile edge counts at k = 97 (one message; a full tile; one past it)"""
    set_path(mr, "tcw")
    rng = random.Random(count)
    N = rng.getrandbits(3072) | (1 << 3071) | 1
    xs = [rng.randrange(N) for _ in range(count)]
    E = rng.getrandbits(128) | (1 << 127)
    y, st, _ = modexp(torch_cuda, mr, N, xs, E, 96)
    assert st == [0] * count
    assert np.array_equal(y, orc.modexp_batch(mr.ints_to_limbs(xs, 96), E, N, threads=8))


def test_tcw_empty_batch(torch_cuda, mr):
    set_path(mr, "tcw")
    N = (1 << 3071) + 12345
    ctx = mr.RnsContext(N | 1, 96)
    x = torch_cuda.empty((0, 96), dtype=torch_cuda.int32, device="cuda")
    ctx.modexp(x, torch_cuda.empty_like(x), 65537)
    torch_cuda.cuda.synchronize()


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("half_bits", [3072, 4096])
def test_tcw_crt_decrypt_vs_oracle(torch_cuda, mr, orc, half_bits, path):
    """CRT decryption of 6144- / 8192-bit keys: both half ladders (k = 97 / 129) in one tcw launch (two contexts),
    then the positional recombination; random coprime odd p, q (Garner's definition O7 needs no primality), ragged
    batch of 300 with edge inputs, every output vs the oracle"""
    set_path(mr, path)
    rng = random.Random(half_bits + 5)
    while True:
        p = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        q = rng.getrandbits(half_bits) | (3 << (half_bits - 2)) | 1
        if p != q and math.gcd(p, q) == 1:
            break
    n, H = p * q, half_bits // 32
    dp, dq = rng.getrandbits(160) | 1, rng.getrandbits(160) | 1
    qinv = pow(q, -1, p)
    cs = [0, 1, n - 1, p, q, 2 * p, 3 * q] + [rng.randrange(n) for _ in range(292)] + [n + 1]
    key = mr.RsaPrivateKey(p, q, dp, dq, qinv)
    c = dev(torch_cuda, mr.ints_to_limbs(cs, 2 * H))
    m = torch_cuda.empty_like(c)
    st = torch_cuda.full((len(cs),), -1, dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=st)
    torch_cuda.cuda.synchronize()
    assert host(st).view(np.int32).tolist() == [0] * 299 + [5]
    ref = orc.crt_decrypt_batch(mr.ints_to_limbs(cs[:299], 2 * H), p, q, dp, dq, qinv, H, threads=8)
    got = host(m)
    assert np.array_equal(got[:299], ref) and not got[299].any()


def test_tcw_paths_identical_full_exponent(torch_cuda, mr):
    """tensor path and IMAD wide kernel produce identical bytes on 1,000 messages with a full 3072-bit exponent"""
    rng = random.Random(3)
    N = rng.getrandbits(3072) | (1 << 3071) | 1
    xs = [rng.randrange(N) for _ in range(1000)]
    E = rng.getrandbits(3072) | (1 << 3071)
    set_path(mr, "tcw")
    a, _, _ = modexp(torch_cuda, mr, N, xs, E, 96)
    set_path(mr, "imad_wide")
    b, _, _ = modexp(torch_cuda, mr, N, xs, E, 96)
    assert np.array_equal(a, b)
    for i in (0, 1, 499, 998, 999):
        assert int.from_bytes(a[i].tobytes(), "little") == pow(xs[i], E, N)


_MULTI_JOB = r"""
import random, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1305_3699_b200 as mr
for bits in (3072, 4096, 8192, 16128):
    rng = random.Random(bits + 3)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [rng.randrange(N) for _ in range(1100)]
    E = rng.getrandbits(96) | (1 << 95)
    ctx = mr.RnsContext(N, L)
    x = torch.from_numpy(mr.ints_to_limbs(xs, L).view(np.int32)).cuda()
    y = torch.empty_like(x)
    ctx.modexp(x, y, E)
    got = mr.limbs_to_ints(y.cpu().numpy())
    assert got == [pow(v, E, N) for v in xs], bits
print("multi-job ok")
"""


def test_tcw_several_jobs_per_cta(torch_cuda):
    """the persistent job loop: 1,100 messages = 9 tile-jobs on a grid capped at 2 CTAs (MR_RNS_MAX_SMS=2, read once
    per process: a subprocess), so every CTA runs several jobs back to back through the same barrier phases"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MR_RNS_MAX_SMS="2")
    r = subprocess.run([sys.executable, "-c", _MULTI_JOB.format(root=root)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "multi-job ok" in r.stdout, r.stderr[-2000:]
