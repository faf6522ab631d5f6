"""One wide-operand launch for profiling: 4,736 messages (default) over a random 8192-bit modulus (k = 257).
    python tools/wide_probe.py [bits] [exponent_bits] [messages]"""
import random
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1305_3699_b200 as mr  # noqa: E402
import synth  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ebits = int(sys.argv[2]) if len(sys.argv) > 2 else 64
rng = random.Random(bits)
N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
limbs = (bits + 31) // 32
ctx = mr.RnsContext(N, limbs)
cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 4736
xs = synth.messages(N, cnt, 1, limbs)
x = torch.from_numpy(xs.view(np.int32)).cuda()
y = torch.empty_like(x)
E = rng.getrandbits(ebits) | (1 << (ebits - 1))
for _ in range(2):
    ctx.modexp(x, y, E)
torch.cuda.synchronize()
print("ok", ctx.k)
