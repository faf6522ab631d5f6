"""One tensor-core wide launch for ncu: python tools/tcw_one.py BITS EBITS COUNT (EBITS 17 = e 65537); two
launches (the first warms up; profile with -s 1 -c 1)."""
import os
import random
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3699_b200 as mr  # noqa: E402

bits, ebits, count = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = random.Random(bits)
N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
L = bits // 32
E = 65537 if ebits == 17 else rng.getrandbits(ebits) | (1 << (ebits - 1))
xs = np.tile(mr.ints_to_limbs([rng.randrange(N) for _ in range(256)], L), (count // 256, 1))
ctx = mr.RnsContext(N, L)
x = torch.from_numpy(np.ascontiguousarray(xs).view(np.int32)).cuda()
y = torch.empty_like(x)
for _ in range(2):
    ctx.modexp(x, y, E)
torch.cuda.synchronize()
print("ok", ctx.k)
