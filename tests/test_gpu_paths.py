"""The same parity cases on every ladder path a narrow-k batch can take:

* ``tensor``: the persistent tcgen05 kernel (k_modexp_tc; small batches forced onto it),
* ``lanes``: the small-batch channels-on-threads kernel, one message per CTA (mr_lanes.cu),
* ``imad``: the thread-per-message IMAD-pipe kernel (k_modexp).

The path is chosen in-process with the library's test hooks (mr_internal_set_small_max, mr_internal_set_path),
so every case runs all three on identical inputs; every output is compared with the CPU oracle.  Covers k = 17,
33, 49 and 65 (512- to 2048-bit moduli and CRT halves), ragged counts, edge inputs, out-of-range inputs and
empty batches.
"""
import ctypes
import random

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

PATHS = ["tensor", "lanes", "imad"]


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
    L.mr_internal_set_small_max.argtypes = [ctypes.c_long]
    L.mr_internal_set_path.argtypes = [ctypes.c_int]
    return mr


@pytest.fixture(params=PATHS)
def path(request, mr):
    L = mr.lib()
    name = request.param
    L.mr_internal_set_path(0 if name == "imad" else 1)
    L.mr_internal_set_small_max(1 << 40 if name == "lanes" else 0)
    yield name
    L.mr_internal_set_path(-1)
    L.mr_internal_set_small_max(-1)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("bits,count", [(512, 1), (512, 129), (1024, 256), (1536, 97), (2048, 300)])
def test_modexp_random_moduli(torch_cuda, mr, orc, path, bits, count):
    rng = random.Random(bits * 7 + count)
    N = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
    L = bits // 32
    xs = [rng.randrange(N) for _ in range(count - 1)] + [N - 1]
    ctx = mr.RnsContext(N, L)
    x = dev(torch_cuda, mr.ints_to_limbs(xs, L))
    for E in (65537, rng.getrandbits(bits) | (1 << (bits - 1)), 0, 1):
        y = torch_cuda.empty_like(x)
        ctx.modexp(x, y, E)
        torch_cuda.cuda.synchronize()
        assert np.array_equal(host(y), orc.modexp_batch(mr.ints_to_limbs(xs, L), E, N, threads=8)), (path, E)


def test_c1_all_ops(torch_cuda, mr, orc, keys, path):
    """C1 (RSA-1024, 256 messages): encrypt, full-d decrypt, CRT decrypt, every output."""
    k = keys["rsa1024"]
    n, L = k["n"], 32
    msgs = synth.messages(n, 256, 0x5EEDC001, L, edge=synth.edge_values(n, k["p"], k["q"]))
    ctx = mr.RnsContext(n, L)
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    x = dev(torch_cuda, msgs)
    c, m1, m2 = torch_cuda.empty_like(x), torch_cuda.empty_like(x), torch_cuda.empty_like(x)
    ctx.encrypt(x, c, k["e"])
    ctx.modexp(c, m1, k["d"])
    key.decrypt(c, m2)
    torch_cuda.cuda.synchronize()
    assert np.array_equal(host(c), orc.modexp_batch(msgs, k["e"], n, threads=8))
    assert np.array_equal(host(m1), msgs) and np.array_equal(host(m2), msgs)


def test_crt_edges_and_status(torch_cuda, mr, orc, keys, path):
    """RSA-2048 CRT (k = 33 halves): edge ciphertexts, out-of-range inputs get status 5 and zeros."""
    k = keys["rsa2048"]
    n, p, q = k["n"], k["p"], k["q"]
    edge = [0, 1, 2, n - 1, n - 2, p, q, 2 * p, 3 * q, p * 5, q - 1, p + 1, 0xDEADBEEF]
    cs = synth.messages(n, 77, 99, 64, edge=edge)
    cs[70] = np.frombuffer(n.to_bytes(256, "little"), dtype=np.uint32)              # = N: out of range
    cs[71] = np.frombuffer(((1 << 2048) - 1).to_bytes(256, "little"), dtype=np.uint32)
    key = mr.RsaPrivateKey(p, q, k["dp"], k["dq"], k["qinv"])
    c = dev(torch_cuda, cs)
    m = torch_cuda.empty_like(c)
    st = torch_cuda.zeros(77, dtype=torch_cuda.int32, device="cuda")
    key.decrypt(c, m, d_status=st)
    torch_cuda.cuda.synchronize()
    ok = [i for i in range(77) if i not in (70, 71)]
    ref = orc.crt_decrypt_batch(cs[ok], p, q, k["dp"], k["dq"], k["qinv"], 32, threads=8)
    assert np.array_equal(host(m)[ok], ref)
    s = host(st).view(np.int32)
    assert s[70] == 5 and s[71] == 5 and not host(m)[70].any() and not host(m)[71].any()
    assert all(s[i] == 0 for i in ok)


def test_k65_and_empty(torch_cuda, mr, orc, keys, path):
    """2048-bit modulus (k = 65: the CTA-pair tensor kernel, or the small-batch kernel), and count = 0."""
    k = keys["rsa2048"]
    n = k["n"]
    xs = synth.messages(n, 65, 0x5EEDC065, 64, edge=synth.edge_values(n, k["p"], k["q"]))
    ctx = mr.RnsContext(n)
    assert ctx.k == 65
    x = dev(torch_cuda, xs)
    y = torch_cuda.empty_like(x)
    ctx.modexp(x, y, k["d"])
    torch_cuda.cuda.synchronize()
    assert np.array_equal(host(y), orc.modexp_batch(xs, k["d"], n, threads=8))
    ctx.modexp(x[:0], y[:0], k["e"])
    torch_cuda.cuda.synchronize()
