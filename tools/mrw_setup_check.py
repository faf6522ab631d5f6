"""Check the wide Miller-Rabin setup rows (mr_internal_mr_wide_setup) against their definitions for a few candidates."""
import ctypes, os, random, sys
import numpy as np, torch
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import paper_1305_3699_b200 as mr
L_ = mr.lib()
k = 257
P32 = ctypes.POINTER(ctypes.c_uint32)
L_.mr_internal_base_table.restype = ctypes.c_int
n = L_.mr_internal_base_table(k, None, 0, None)
flat = np.zeros(n, dtype=np.uint32); primes = np.zeros(2 * k, dtype=np.uint32)
L_.mr_internal_base_table(k, flat.ctypes.data_as(P32), n, primes.ctypes.data_as(P32))
primes = [int(p) for p in primes]
B, Bp = primes[:k], primes[k:]
M = 1
for m in B: M *= m
Mp = 1
for m in Bp: Mp *= m
W = 1 << 32
rng = random.Random(3)
bits = 4160
Lm = (bits + 31) // 32
ns = [rng.getrandbits(bits) | (1 << (bits - 1)) | 1 for _ in range(3)]
cnt = len(ns)
d_n = torch.from_numpy(mr.ints_to_limbs(ns, Lm).view(np.int32)).cuda()
words = 8 * k + 9
d_pcw = torch.zeros(words * cnt, dtype=torch.int32, device='cuda')
d_v = torch.zeros(cnt, dtype=torch.uint8, device='cuda')
rc = L_.mr_internal_mr_wide_setup(ctypes.c_void_p(d_n.data_ptr()), ctypes.c_size_t(Lm), ctypes.c_size_t(cnt), k,
                                  ctypes.c_void_p(d_pcw.data_ptr()), ctypes.c_void_p(d_v.data_ptr()), 0)
print('rc', rc)
pc = d_pcw.cpu().numpy().view(np.uint32).reshape(words, cnt)
for q, N in enumerate(ns):
    errs = []
    for i in [0, 1, k - 1]:
        m = B[i]; Mi = M // m
        sg = (-pow(N * Mi, -1, m)) % m
        if int(pc[0 + i, q]) != sg * W * W % m: errs.append(('sig', i))
    for j in [0, 1, k - 1]:
        m = Bp[j]; lam = pow(Mp // m, -1, m)
        c2 = N * pow(M, -1, m) * lam % m
        if int(pc[k + j, q]) != c2 * W % m: errs.append(('c2', j))
    R2 = M * M % N
    for c in [0, 1, k - 1, k, 2 * k - 1]:
        m = (B + Bp)[c]
        want = R2 % m if c < k else R2 % m * pow(Mp // m, -1, m) % m
        if int(pc[2 * k + c, q]) != want: errs.append(('r2', c, int(pc[2 * k + c, q]), want))
    if int(pc[2 * k + 2 * k, q]) != R2 % W: errs.append('r2r')
    if int(pc[4 * k + 1, q]) != N * pow(M, -1, W) % W: errs.append('nminv')
    s = ((N - 1) & -(N - 1)).bit_length() - 1
    if int(pc[4 * k + 2, q]) != s: errs.append('s')
    d = (N - 1) >> s
    dd = sum(int(pc[4 * k + 4 + l, q]) << (32 * l) for l in range(k))
    if dd != d: errs.append('d')
    print(q, 'live', int(pc[4 * k + 3, q]), errs[:6])
