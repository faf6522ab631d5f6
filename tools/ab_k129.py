"""A/B probe for b-bit operands (default 4096, k = 129): b-bit modexp with a full-length exponent, RSA-b
encryption (e = 65537) and RSA-2b CRT decryption (b-bit halves).  Prints one line per workload with the
rate and a sampled bit-exact check against Python's pow.  MR_RNS_WIDE_MIN=k' moves every k >= k' (>= 97)
onto the wide-operand kernel (default 97; 999: the per-k IMAD kernels).
    python tools/ab_k129.py [b]"""
import math
import os
import random
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3699_b200 as mr  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


rng = random.Random(129)
tag = os.environ.get("MR_RNS_WIDE_MIN", "97")
BITS = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = BITS // 32
# BITS-bit modexp, full exponent
N = rng.getrandbits(BITS) | (1 << BITS - 1) | 1
ctx = mr.RnsContext(N, L)
cnt = int(os.environ.get("AB_CNT_EXP", 8192))
x = torch.from_numpy(synth.messages(N, cnt, 1, L).view(np.int32)).cuda()
y = torch.empty_like(x)
E = rng.getrandbits(BITS) | (1 << BITS - 1)
t = timed(lambda: ctx.modexp(x, y, E), 2)
xs, ys = mr.limbs_to_ints(x.cpu().numpy()), mr.limbs_to_ints(y.cpu().numpy())
ok = all(pow(xs[i], E, N) == ys[i] for i in (0, 1, cnt // 2, cnt - 1))
print(f"wide_min={tag} k={ctx.k} modexp{BITS}_fullexp {cnt / t:.0f}/s ok={ok}")
# RSA-BITS encryption
cnt = 65536
x = torch.from_numpy(synth.messages(N, cnt, 2, L).view(np.int32)).cuda()
y = torch.empty_like(x)
t = timed(lambda: ctx.encrypt(x, y, 65537), 5)
xs, ys = mr.limbs_to_ints(x.cpu().numpy()), mr.limbs_to_ints(y.cpu().numpy())
ok = all(pow(xs[i], 65537, N) == ys[i] for i in (0, 1, cnt // 2, cnt - 1))
print(f"wide_min={tag} rsa{BITS}_encrypt {cnt / t:.0f}/s ok={ok}")
# RSA-8192 CRT decryption
# coprime odd halves (the CRT path needs only gcd(p, q) = 1: Garner, HAC 14.71)
while True:
    p = rng.getrandbits(BITS) | (3 << BITS - 2) | 1
    q = rng.getrandbits(BITS) | (3 << BITS - 2) | 1
    if math.gcd(p, q) == 1:
        break
n = p * q
dp, dq = rng.getrandbits(BITS) % p, rng.getrandbits(BITS) % q
key = mr.RsaPrivateKey(p, q, dp, dq, pow(q, -1, p), L)
cnt = int(os.environ.get("AB_CNT_CRT", BITS))
c = torch.from_numpy(synth.messages(n, cnt, 3, 2 * L).view(np.int32)).cuda()
m = torch.empty_like(c)
t = timed(lambda: key.decrypt(c, m), 2)
cs, ms = mr.limbs_to_ints(c.cpu().numpy()), mr.limbs_to_ints(m.cpu().numpy())
ok = all(ms[i] < n and ms[i] % p == pow(cs[i], dp, p) and ms[i] % q == pow(cs[i], dq, q)
         for i in (0, 1, cnt // 2, cnt - 1))
print(f"wide_min={tag} rsa{2 * BITS}_crt {cnt / t:.0f}/s ok={ok}")
