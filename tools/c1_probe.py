"""C1 probe (BASELINE configs[0]: RSA-1024, 256 seeded messages, encrypt e = 65537, decrypt with full d and with CRT):
throughput of each (CUDA events, best of 5) and bit-exactness vs the oracle.  Usable under ncu and with MR_RNS_LIB.
    python tools/c1_probe.py [reps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402
import paper_1305_3699_b200 as mr  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
k = bench.load_key("rsa1024")
n = k["n"]
msgs = synth.messages(n, 256, 0x5EEDC001, 32, edge=synth.edge_values(n, k["p"], k["q"]))
ctx = mr.RnsContext(n, 32)
priv = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
x = torch.from_numpy(msgs.view(np.int32)).cuda()
c, m1, m2 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)


def best(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


t_enc = best(lambda: ctx.encrypt(x, c, k["e"]))
t_dec = best(lambda: ctx.modexp(c, m1, k["d"]))
t_crt = best(lambda: priv.decrypt(c, m2))
ok = bool(np.array_equal(c.cpu().numpy().view(np.uint32), oracle.modexp_batch(msgs, k["e"], n, threads=os.cpu_count()))
          and np.array_equal(m1.cpu().numpy().view(np.uint32), msgs) and np.array_equal(m2.cpu().numpy().view(np.uint32), msgs))
print(f"C1 encrypt {256 / t_enc:,.0f}/s  decrypt_full_d {256 / t_dec:,.0f}/s ({t_dec * 1e6:.0f} us)  "
      f"decrypt_crt {256 / t_crt:,.0f}/s  bit_exact {ok}", flush=True)
