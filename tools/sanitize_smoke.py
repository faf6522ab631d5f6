"""compute-sanitizer smoke runs of every hand-written kernel family at C1-like sizes (
SURVEY §4 T5).  One case per process:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_smoke.py <case>

Cases (each checks its outputs against Python's pow / the property it computes):
  crt33     RSA-2048 CRT decryption, k = 33 tensor kernel + k_combine, 600 messages on a grid capped at
            2 SMs (MR_RNS_MAX_SMS=2) so the split hand-over schedule runs
  pair65    2048-bit modexp, k = 65 CTA-pair tensor kernel, 700 messages on 2 SMs (split schedule)
  mr33      Miller-Rabin, 1024-bit candidates, k_mr_setup / k_mr_rounds_tc / k_mr_final, 300 candidates
  wide97    RSA-3072 encryption on the wide-operand kernel (k = 97), 40 messages
  imad33    RSA-1024 modexp on the IMAD-path kernel (MR_RNS_IMAD_ONLY=1), 200 messages
  drbg      Hash_DRBG generate + FIPS 140-2 health kernel
  keygen    mr_rsa_keygen_batch_drbg, 2 RSA-1024 keys
  tcw257    8192-bit modexp on the tensor-core wide kernel (k = 257, one tile per CTA), 20 messages, 24-bit E
  tcw505    16,128-bit modexp on the tensor-core wide kernel (k = 505, 64-message tiles), 10 messages, 24-bit E
  lanes33   RSA-1024 modexp on the small-batch lanes kernel (k = 33, one message per CTA), 40 messages, 200-bit E
"""
import os
import random
import sys

CASE = sys.argv[1] if len(sys.argv) > 1 else "crt33"
if CASE in ("crt33", "pair65"):
    os.environ.setdefault("MR_RNS_MAX_SMS", "2")
if CASE == "imad33":
    os.environ["MR_RNS_IMAD_ONLY"] = "1"

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3699_b200 as mr  # noqa: E402

torch.cuda.set_device(0)
rng = random.Random(1)


def dev(rows):
    return torch.from_numpy(np.ascontiguousarray(rows, dtype=np.uint32).view(np.int32)).cuda()


def ints(t):
    return [int.from_bytes(r.tobytes(), "little") for r in t.cpu().numpy().view(np.uint32)]


def rand_prime(bits):
    import sympy
    return sympy.randprime(3 << (bits - 2), 1 << bits)


if CASE == "crt33" or CASE == "pair65":
    bits = 2048
    p, q = rand_prime(1024), rand_prime(1024)
    if p < q:
        p, q = q, p
    n, e = p * q, 65537
    d = pow(e, -1, (p - 1) * (q - 1))
    cnt = 600 if CASE == "crt33" else 700
    xs = [rng.randrange(n) for _ in range(cnt)]
    x = dev(mr.ints_to_limbs(xs, 64))
    y = torch.empty_like(x)
    if CASE == "crt33":
        key = mr.RsaPrivateKey(p, q, d % (p - 1), d % (q - 1), pow(q, -1, p))
        key.decrypt(x, y)
        E = d
    else:
        ctx = mr.RnsContext(n)
        assert ctx.k == 65
        E = rng.getrandbits(160) | 1
        ctx.modexp(x, y, E)
    torch.cuda.synchronize()
    got = ints(y)
    assert all(got[i] == pow(xs[i], E, n) for i in range(cnt)), CASE
elif CASE == "mr33":
    import sympy
    cands = [rand_prime(1024) if i % 3 == 0 else (rng.getrandbits(1024) | (3 << 1022) | 1) for i in range(300)]
    R = 3
    bases = [[rng.randrange(2, c - 1) for _ in range(R)] for c in cands]
    dn = dev(mr.ints_to_limbs(cands, 32))
    db = dev(np.stack([mr.ints_to_limbs(b, 32) for b in bases]).reshape(len(cands), R * 32))
    v = torch.zeros(len(cands), dtype=torch.uint8, device="cuda")
    w = torch.zeros(len(cands), dtype=torch.int16, device="cuda")
    s = torch.zeros(len(cands), dtype=torch.int32, device="cuda")
    mr.mr_miller_rabin_batch(dn, 32, len(cands), db, R, v, w, s)
    torch.cuda.synchronize()
    vv = v.cpu().tolist()
    assert all((vv[i] == mr.MR_PROBABLY_PRIME) == sympy.isprime(c) for i, c in enumerate(cands) if vv[i] != mr.MR_FACTOR)
elif CASE in ("wide97", "imad33", "tcw257", "tcw505", "lanes33"):
    bits = {"wide97": 3072, "imad33": 1024, "tcw257": 8192, "tcw505": 16128, "lanes33": 1024}[CASE]
    n = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    cnt = {"wide97": 40, "imad33": 200, "tcw257": 20, "tcw505": 10, "lanes33": 40}[CASE]
    xs = [rng.randrange(n) for _ in range(cnt)]
    E = 65537 if CASE == "wide97" else (0xB5A3F1 if CASE.startswith("tcw") else rng.getrandbits(200) | 1)
    ctx = mr.RnsContext(n)
    x = dev(mr.ints_to_limbs(xs, bits // 32))
    y = torch.empty_like(x)
    ctx.modexp(x, y, E)
    torch.cuda.synchronize()
    got = ints(y)
    assert all(got[i] == pow(xs[i], E, n) for i in range(cnt)), CASE
elif CASE == "drbg":
    g = mr.Drbg(bytes(range(32)), bytes(16), b"san", streams=16)
    out = torch.empty((16, 2500 * 4), dtype=torch.uint8, device="cuda")
    g.generate(out, 2500 * 4)
    blocks = out.reshape(64, 2500)
    stats = torch.zeros((64, 16), dtype=torch.int32, device="cuda")
    mr.fips_health(blocks, stats)
    torch.cuda.synchronize()
    assert int((stats[:, 0] > 9725).sum()) >= 60
elif CASE == "keygen":
    g = mr.Drbg(bytes(range(32)), bytes(16), b"san-kg", streams=8)
    outs = [torch.zeros((2, 32 if f in ("n", "d") else 16), dtype=torch.int32, device="cuda")
            for f in ("n", "p", "q", "d", "dp", "dq", "qinv")]
    mr.mr_rsa_keygen_batch_drbg(g, 2, 1024, 65537, 3, *outs)
    torch.cuda.synchronize()
    n0, p0, q0 = ints(outs[0])[0], ints(outs[1])[0], ints(outs[2])[0]
    assert n0 == p0 * q0
else:
    raise SystemExit(f"unknown case {CASE}")
print(f"sanitize_smoke {CASE}: ok", flush=True)
