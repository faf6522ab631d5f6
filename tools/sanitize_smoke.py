import sys, numpy as np, torch, random
sys.path.insert(0, '/root/repo')
import paper_1305_3699_b200 as mr
torch.cuda.set_device(0)
def run(N, xs, E, limbs):
    ctx = mr.RnsContext(N, limbs)
    x = torch.from_numpy(mr.ints_to_limbs(xs, limbs).view(np.int32)).cuda()
    y = torch.empty_like(x)
    ctx.modexp(x, y, E)
    torch.cuda.synchronize()
    return [int.from_bytes(r.tobytes(), 'little') for r in y.cpu().numpy().view(np.uint32)], ctx.k
rng = random.Random(1)
for bits, cnt in ((1024, 300), (2048, 600), (8192, 20)):
    N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
    xs = [rng.randrange(N) for _ in range(cnt)]
    E = rng.getrandbits(64) | 1
    y, k = run(N, xs, E, (bits + 31) // 32)
    assert all(y[i] == pow(xs[i], E, N) for i in range(cnt)), bits
    print("ok", bits, k, flush=True)
