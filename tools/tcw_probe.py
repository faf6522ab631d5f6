"""Probe of the tensor-core wide kernel (k = 97 / 129 / 257, mr_tcw.cuh): parity vs Python pow on ragged batches, then
throughput of RSA-3072 / 4096 encryption and full-exponent modexp (tcw vs the IMAD wide kernel).
    python tools/tcw_probe.py [quick]"""
import os
import random
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1305_3699_b200 as mr  # noqa: E402


def run(N, L, xs, E):
    ctx = mr.RnsContext(N, L)
    x = torch.from_numpy(mr.ints_to_limbs(xs, L).view(np.int32)).cuda()
    y = torch.empty_like(x)
    st = torch.zeros(len(xs), dtype=torch.int32, device="cuda")
    ctx.modexp(x, y, E, d_status=st)
    torch.cuda.synchronize()
    return mr.limbs_to_ints(y.cpu().numpy()), st.cpu().tolist(), ctx


ok_all = True
for bits in (3072, 4096, 8192, 16128):
    rng = random.Random(bits)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    xs = [0, 1, 2, N - 1, N - 2] + [rng.randrange(N) for _ in range(290)] + [N + 5]
    for E in (3, 65537, rng.getrandbits(200) | (1 << 199)):
        t0 = time.time()
        y, st, ctx = run(N, L, xs, E)
        ref = [pow(v, E, N) for v in xs[:-1]]
        bad = [i for i in range(len(ref)) if y[i] != ref[i]]
        ok = not bad and st[-1] == 5 and y[-1] == 0
        ok_all &= ok
        print(f"bits={bits} k={ctx.k} E.bits={E.bit_length()} ok={ok} bad={len(bad)} first_bad={bad[:5]} st_last={st[-1]} ({time.time()-t0:.1f}s)", flush=True)
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    sys.exit(0 if ok_all else 1)
for bits, E in ((3072, 65537), (4096, 65537), (8192, 65537), (16128, 65537), (3072, None), (4096, None), (8192, None), (16128, None)):
    rng = random.Random(bits + 7)
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    L = bits // 32
    E = E or (rng.getrandbits(bits) | (1 << (bits - 1)))
    count = 9472 if bits == 16128 else 18944 if bits == 8192 else 65536 if E == 65537 else 37888   # 8192 / 16128: one job per SM
    xs = np.ascontiguousarray(mr.ints_to_limbs([rng.randrange(N) for _ in range(256)], L))
    xs = np.tile(xs, (count // 256, 1))
    ctx = mr.RnsContext(N, L)
    x = torch.from_numpy(xs.view(np.int32)).cuda()
    y = torch.empty_like(x)
    ctx.modexp(x, y, E)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.modexp(x, y, E)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3e3
    print(f"throughput bits={bits} E.bits={E.bit_length()} count={count}: {count / t:,.0f} modexps/s ({t*1e3:.2f} ms)", flush=True)
sys.exit(0 if ok_all else 1)
