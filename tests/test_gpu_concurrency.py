"""Concurrent use of one context / key from several streams and host threads (include/mr_rns.h:
"Contexts ... may be used concurrently from any host thread or stream").

The persistent tensor-core kernel's split schedule hands a job's state from one CTA to
another through a flag.  Two such launches running at once each see only part of the SMs; the kernel
numbers its CTAs in start order (a ticket) so a CTA only waits for one that has already started.  These
tests run two full-size split launches concurrently on two streams, and several host threads over one
context; every output is checked by the round trip enc(dec(c)) = c, sampled outputs against the oracle.
They also cover the bounded program cache: more distinct exponents than the cache holds.
"""
import threading

import numpy as np
import pytest

import synth

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


@pytest.mark.parametrize("counts", [(75777, 38016), (65536 + 128, 65536 + 128)])
def test_two_streams_split_schedule(torch_cuda, mr, orc, keys, counts):
    torch = torch_cuda
    k = keys["rsa2048"]
    n = k["n"]
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    ctx = mr.RnsContext(n)
    cs = [synth.messages(n, c, 0x5EEDC2A0 + i, 64) for i, c in enumerate(counts)]
    cd = [dev(torch, c) for c in cs]
    md = [torch.empty_like(c) for c in cd]
    streams = [torch.cuda.Stream() for _ in counts]
    torch.cuda.synchronize()
    for _ in range(2):                              # twice: the second pair overlaps the first's tail
        for c, m, s in zip(cd, md, streams):
            with torch.cuda.stream(s):
                key.decrypt(c, m, stream=s)
    torch.cuda.synchronize()
    for c, m, cs_ in zip(cd, md, cs):
        c2 = torch.empty_like(c)
        ctx.encrypt(m, c2, k["e"])
        torch.cuda.synchronize()
        assert torch.equal(c, c2)
        idx = [0, 1, 127, 128, len(cs_) // 2, len(cs_) - 1]
        ref = orc.crt_decrypt_batch(cs_[idx], k["p"], k["q"], k["dp"], k["dq"], k["qinv"], 32, threads=8)
        assert np.array_equal(host(m)[idx], ref)


def test_pair_mode_two_streams(torch_cuda, mr, orc, keys):
    """k = 65 CTA-pair kernel (2048-bit modulus) with a split geometry, two streams at once."""
    torch = torch_cuda
    k = keys["rsa2048"]
    n = k["n"]
    ctx = mr.RnsContext(n)
    assert ctx.k == 65
    count = 149 * 256 + 77
    xs = [synth.messages(n, count, 0x5EEDC2B0 + i, 64) for i in range(2)]
    xd = [dev(torch, x) for x in xs]
    yd = [torch.empty_like(x) for x in xd]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for x, y, s in zip(xd, yd, streams):
        with torch.cuda.stream(s):
            ctx.modexp(x, y, k["d"], stream=s)
    torch.cuda.synchronize()
    for x, y, xh in zip(xd, yd, xs):
        z = torch.empty_like(x)
        ctx.modexp(y, z, k["e"])
        torch.cuda.synchronize()
        assert torch.equal(x, z)
        idx = [0, 255, 256, count // 2, count - 1]
        assert np.array_equal(host(y)[idx], orc.modexp_batch(xh[idx], k["d"], n, threads=8))


def test_host_threads_share_context(torch_cuda, mr, orc, keys):
    """4 host threads, each on its own stream, each with its own exponents on ONE context: 80 distinct
    exponents in total, more than the 64-program cache holds (the rest run as stream-ordered transient
    programs); every output vs the oracle."""
    torch = torch_cuda
    k = keys["rsa1024"]
    n = k["n"]
    ctx = mr.RnsContext(n)
    xs = synth.messages(n, 300, 0x5EEDC2C0, 32)
    errors = []

    def worker(t):
        try:
            s = torch.cuda.Stream()
            x = dev(torch, xs)
            for j in range(20):
                E = (1 << (40 + 7 * t + j)) + 2 * j + 1
                y = torch.empty_like(x)
                with torch.cuda.stream(s):
                    ctx.modexp(x, y, E, stream=s)
                s.synchronize()
                sub = [0, 1, 150, 299]
                if not np.array_equal(host(y)[sub], orc.modexp_batch(xs[sub], E, n)):
                    errors.append((t, j))
        except Exception as ex:                      # surface in the main thread
            errors.append(repr(ex))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:4]


def test_binding_rejects_bad_buffers(torch_cuda, mr, keys):
    """wrong dtype, width or size never reaches the kernels."""
    torch = torch_cuda
    k = keys["rsa1024"]
    ctx = mr.RnsContext(k["n"])
    x = torch.zeros((8, 32), dtype=torch.int32, device="cuda")
    for bad in (torch.zeros((8, 32), dtype=torch.int64, device="cuda"), torch.zeros((8, 31), dtype=torch.int32,
                device="cuda"), torch.zeros(8 * 32, dtype=torch.int32, device="cuda"),
                torch.zeros((4, 32), dtype=torch.int32, device="cuda")):
        with pytest.raises(mr.MrError) as e:
            ctx.modexp(x, bad, 65537, count=8)
        assert e.value.code == mr.MR_ERR_ARG
    info = mr.mr_rns_ctx_info(ctx.handle)
    assert info["k"] == 33 and 1024 <= info["max_modulus_bits"] < 33 * 32 and info["modulus_bits"] == 1024


@pytest.mark.parametrize("case", ["crt33", "pair65", "mr33", "wide97", "imad33", "drbg", "keygen"])
def test_sanitize_smoke_cases_plain(torch_cuda, case):
    """the compute-sanitizer smoke cases (tools/sanitize_smoke.py) without the sanitizer: crt33 / pair65 run
    the split schedule on a grid capped at 2 SMs (MR_RNS_MAX_SMS), i.e. every hand-over crosses CTAs."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_smoke.py"), case], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and f"sanitize_smoke {case}: ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
