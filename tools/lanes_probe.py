"""One C1 full-d decryption batch (256 messages) on a chosen ladder path (argv[1]: lanes | tensor), for ncu."""
import ctypes
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
L.mr_internal_set_small_max(1 << 40 if sys.argv[1] == "lanes" else 0)
k = bench.load_key("rsa1024")
ctx = mr.RnsContext(k["n"], 32)
xs = synth.messages(k["n"], int(sys.argv[2]) if len(sys.argv) > 2 else 256, 0x5EED5A, 32)
x = torch.from_numpy(xs.view(np.int32)).cuda()
y = torch.empty_like(x)
for _ in range(2):
    ctx.modexp(x, y, k["d"])
torch.cuda.synchronize()
print("ok")
