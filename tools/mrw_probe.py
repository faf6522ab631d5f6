import os, random, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.path.join(os.environ.get('GRAFT_REPO_ROOT', '/root/repo')))
import paper_1305_3699_b200 as mr
import sympy
rng = random.Random(7)
for bits in [int(b) for b in (sys.argv[1:] or ["4160"])]:
    L = (bits + 31) // 32
    ns = []
    p = sympy.nextprime(rng.getrandbits(bits) | (1 << (bits - 1)))
    ns.append(p)                                     # prime
    ns.append(p * 3 if (p * 3).bit_length() <= 32 * L else p - 2)  # composite-ish
    while len(ns) < 40:
        ns.append(rng.getrandbits(bits) | (1 << (bits - 1)) | 1)
    R = 3
    bases = [[rng.randrange(2, n - 1) for _ in range(R)] for n in ns]
    d_n = torch.from_numpy(mr.ints_to_limbs(ns, L).view(np.int32)).cuda()
    d_b = torch.from_numpy(np.ascontiguousarray(np.stack([mr.ints_to_limbs(b, L) for b in bases])).view(np.int32)).cuda()
    v = torch.zeros(len(ns), dtype=torch.uint8, device='cuda'); w = torch.zeros(len(ns), dtype=torch.int16, device='cuda')
    s = torch.zeros(len(ns), dtype=torch.int32, device='cuda')
    mr.mr_miller_rabin_batch(d_n, L, len(ns), d_b, R, v, w, s)
    torch.cuda.synchronize()
    v = v.cpu().tolist(); w = w.cpu().tolist(); s = s.cpu().tolist()
    def ref(n, bs):
        d, sh = n - 1, 0
        while d % 2 == 0: d //= 2; sh += 1
        for r, a in enumerate(bs):
            y = pow(a, d, n)
            if y in (1, n - 1): continue
            for _ in range(sh - 1):
                y = y * y % n
                if y == n - 1: break
            else:
                return 0, r
        return 1, -1
    rv = [ref(n, b) for n, b in zip(ns, bases)]
    bad = [i for i in range(len(ns)) if (v[i], w[i]) != rv[i]]
    print(bits, 'ok' if not bad else f'BAD {bad[:5]} got {[(v[i], w[i]) for i in bad[:3]]} want {[rv[i] for i in bad[:3]]}', set(s), flush=True)
