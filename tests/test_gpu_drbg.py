"""GPU parity of the DRBG and FIPS 140-2 health-test kernels against
the oracle (oracle/drbg.py): every output byte and every statistic, bit-exact."""
import numpy as np
import pytest

from oracle import drbg

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


def test_drbg_streams_vs_oracle(torch_cuda, mr):
    """37 streams, successive requests of 100, 65,536 (the per-request maximum), 0 (state update only),
    33 and 32 bytes: every byte of every stream equals SP 800-90A Hash_DRBG in the oracle."""
    e, n, p = bytes(range(40)), bytes(range(100, 116)), b"mr-trng"
    streams, sizes = 37, [100, 65536, 0, 33, 32]
    g = mr.Drbg(e, n, p, streams)
    refs = [drbg.HashDrbg(e, n, drbg.stream_pers(p, s)) for s in range(streams)]
    for nb in sizes:
        out = torch_cuda.zeros(streams * nb, dtype=torch_cuda.uint8, device="cuda")
        g.generate(out if nb else None, nb)
        torch_cuda.cuda.synchronize()
        got = out.cpu().numpy().reshape(streams, nb) if nb else None
        for s in range(streams):
            want = refs[s].generate(nb)
            if nb:
                assert got[s].tobytes() == want, (nb, s)


def test_drbg_argument_rules(torch_cuda, mr):
    with pytest.raises(mr.MrError):
        mr.Drbg(bytes(31), bytes(16))                      # entropy below 256 bits
    with pytest.raises(mr.MrError):
        mr.Drbg(bytes(32), bytes(15))                      # nonce below 128 bits
    g = mr.Drbg(bytes(32), bytes(16), streams=2)
    with pytest.raises(mr.MrError):
        g.generate(torch_cuda.zeros(2 * 65537, dtype=torch_cuda.uint8, device="cuda"), 65537)


def test_fips_health_vs_oracle(torch_cuda, mr):
    """constructed blocks (all zeros, alternating, monobit and long-run edges) and 300 DRBG blocks: the
    16 statistics per block equal the oracle's counts; verdict bits equal the oracle's verdicts."""
    rng = np.random.default_rng(9)
    blocks = [bytes(2500), bytes([0x55]) * 2500, bytes([0xFF]) * 2500]
    for ones in (9725, 9726, 10274, 10275):
        bits = np.zeros(20000, dtype=np.uint8)
        bits[rng.choice(20000, ones, replace=False)] = 1
        blocks.append(np.packbits(bits).tobytes())
    for ln in (25, 26, 31, 33, 64):
        bits = np.tile(np.array([0, 1], dtype=np.uint8), 10000)
        bits[1000:1000 + ln] = 1
        bits[999] = 0
        bits[1000 + ln] = 0
        blocks.append(np.packbits(bits).tobytes())
    d = drbg.HashDrbg(b"\x07" * 32, b"\x08" * 16, b"health")
    data = d.hashgen(2500 * 300)
    blocks += [data[i * 2500:(i + 1) * 2500] for i in range(300)]
    arr = np.frombuffer(b"".join(blocks), dtype=np.uint8).reshape(len(blocks), 2500)
    db = torch_cuda.from_numpy(arr.copy()).cuda()
    ds = torch_cuda.zeros((len(blocks), 16), dtype=torch_cuda.int32, device="cuda")
    mr.fips_health(db, ds)
    torch_cuda.cuda.synchronize()
    st = ds.cpu().numpy().view(np.uint32)
    for i, b in enumerate(blocks):
        h = drbg.health(b)
        assert st[i, 0] == h["ones"] and st[i, 1] == h["poker_s"]
        assert list(st[i, 2:8]) == list(h["runs"][1]) and list(st[i, 8:14]) == list(h["runs"][0])
        assert st[i, 14] == (1 if h["longest"] >= 26 else 0)
        v = int(h["monobit"]) | int(h["poker"]) << 1 | int(h["runs_ok"]) << 2 | int(h["long_run"]) << 3
        assert st[i, 15] == v, i
