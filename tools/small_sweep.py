"""Small-batch crossover sweep: the same batch on the tensor kernel and on the one-message-per-
CTA kernel (mr_lanes.cu), chosen in-process with mr_internal_set_small_max; CUDA-event time, best of 3, sampled
outputs checked against Python's pow.  Prints one JSON line per (workload, count, path)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_3699_b200 as mr  # noqa: E402
import synth  # noqa: E402

L = mr.lib()
L.mr_internal_set_small_max.argtypes = [ctypes.c_long]
torch.cuda.set_device(0)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


for name, keyname, limbs, op in (("C1 RSA-1024 full-d decrypt", "rsa1024", 32, "d"),
                                 ("RSA-2048 CRT decrypt", "rsa2048", 64, "crt"),
                                 ("RSA-3072 CRT decrypt", "rsa3072", 96, "crt")):
    k = bench.load_key(keyname)
    n = k["n"]
    ctx = mr.RnsContext(n, limbs)
    key = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    for count in (64, 256, 1024, 2048, 4096, 8192):
        xs = synth.messages(n, count, 0x5EED5A, limbs)
        x = torch.from_numpy(xs.view(np.int32)).cuda()
        y = torch.empty_like(x)
        for path in ("tensor", "lanes"):
            L.mr_internal_set_small_max(1 << 40 if path == "lanes" else 0)
            fn = (lambda: ctx.modexp(x, y, k["d"])) if op == "d" else (lambda: key.decrypt(x, y))
            t = timed(fn)
            got = y.cpu().numpy().view(np.uint32)
            ok = all(int.from_bytes(got[i].tobytes(), "little") == pow(int.from_bytes(xs[i].tobytes(), "little"),
                                                                        k["d"], n) for i in (0, count // 2, count - 1))
            print(json.dumps({"workload": name, "count": count, "path": path, "seconds": t, "ops_per_s": count / t,
                              "sample_ok": ok}), flush=True)
L.mr_internal_set_small_max(-1)
