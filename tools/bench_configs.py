"""Secondary measurements of BASELINE.json's other configs (C1, C3, C4, C5) on one GPU.

bench.py measures the headline config (C2).  This script times the others through the same C ABI,
prints one JSON line per point and checks a sample of every point against the CPU oracle:

  C1  RSA-1024, 256 messages: encrypt (e = 65537), decrypt with the full d, CRT decrypt
  C3  RSA-3072: encrypt (k = 97) and CRT decrypt (k = 49 per half), batch sweep
  C4  2048-bit modulus (k = 65), exponents of 1,024 ... 16,128 bits
  C5  Miller-Rabin on seeded 1024-bit candidates (k = 33), 5 rounds, forced and early-exit
  RNG Hash_DRBG (SHA-256) generation and FIPS 140-2 health tests (§8(f) row 4), GB/s
  W   wide operands (§8(f) row 3): 4096-bit (k = 129), 8192-bit (k = 257) and 16,128-bit (k = 505) moduli,
      e = 65537 and a full-length exponent

    python tools/bench_configs.py [--configs C1,C3,C4,C5] [--quick]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def per_mm(k):
    return 2 * k * k + 8 * k + 4


def timed(torch, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return best


def emit(rec):
    print(json.dumps(rec), flush=True)


def peak():
    return bench.peak_imad_eq_per_s(1965.0)


def c1(torch, mr, orc):
    k = bench.load_key("rsa1024")
    n = k["n"]
    msgs = synth.messages(n, 256, 0x5EEDC001, 32, edge=synth.edge_values(n, k["p"], k["q"]))
    ctx = mr.RnsContext(n, 32)
    priv = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    x = torch.from_numpy(msgs.view(np.int32)).cuda()
    c, m1, m2 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    t_enc = timed(torch, lambda: ctx.encrypt(x, c, k["e"]))
    t_dec = timed(torch, lambda: ctx.modexp(c, m1, k["d"]))
    t_crt = timed(torch, lambda: priv.decrypt(c, m2))
    ok = bool(np.array_equal(c.cpu().numpy().view(np.uint32), orc.modexp_batch(msgs, k["e"], n, threads=os.cpu_count()))
              and np.array_equal(m1.cpu().numpy().view(np.uint32), msgs)
              and np.array_equal(m2.cpu().numpy().view(np.uint32), msgs))
    for op, t, mm in (("encrypt", t_enc, bench.sliding_window_mm(k["e"])), ("decrypt_full_d", t_dec, bench.sliding_window_mm(k["d"])),
                      ("decrypt_crt", t_crt, bench.sliding_window_mm(k["dp"]) + bench.sliding_window_mm(k["dq"]))):
        kk = 33 if op != "decrypt_crt" else 17
        emit({"config": "C1", "op": op, "messages": 256, "seconds": t, "ops_per_s": 256 / t,
              "imad_eq_frac": 256 * mm * 2 * per_mm(kk) / t / peak(), "bit_exact_all_256": ok})


def c3(torch, mr, orc, quick):
    k = bench.load_key("rsa3072")
    n = k["n"]
    ctx = mr.RnsContext(n, 96)
    priv = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"])
    # BASELINE configs[2]: the 1K-1M sweep (one GPU here; bench.py --total T --gpus N shards it)
    sizes = [1024, 4096, 16384] if quick else [1024, 4096, 16384, 65536, 262144, 1048576]
    for cnt in sizes:
        msgs = synth.messages(n, cnt, 0x5EEDC003, 96, edge=synth.edge_values(n, k["p"], k["q"]))
        x = torch.from_numpy(msgs.view(np.int32)).cuda()
        c, m = torch.empty_like(x), torch.empty_like(x)
        t_enc = timed(torch, lambda: ctx.encrypt(x, c, k["e"]), reps=2)
        t_dec = timed(torch, lambda: priv.decrypt(c, m), reps=2)
        s = min(cnt, 256)
        ok = bool(np.array_equal(m.cpu().numpy().view(np.uint32), msgs) and np.array_equal(
            c.cpu().numpy().view(np.uint32)[:s], orc.modexp_batch(msgs[:s], k["e"], n, threads=os.cpu_count())))
        mm_dec = bench.sliding_window_mm(k["dp"]) + bench.sliding_window_mm(k["dq"])
        emit({"config": "C3", "messages": cnt, "encrypt_ops_per_s": cnt / t_enc, "decrypt_crt_ops_per_s": cnt / t_dec,
              "encrypt_k": ctx.k, "decrypt_imad_eq_frac": cnt * mm_dec * 2 * per_mm(49) / t_dec / peak(),
              "encrypt_imad_eq_frac": cnt * bench.sliding_window_mm(k["e"]) * 2 * per_mm(97) / t_enc / peak(),
              "bit_exact": ok, "checked": f"decrypt(encrypt(m)) = m for all {cnt}; encrypt vs oracle on {s}"})


def c4(torch, mr, orc, quick):
    k = bench.load_key("rsa2048")
    n = k["n"]
    ctx = mr.RnsContext(n, 64)
    for ell in ([1024, 16128] if quick else [17, 1024, 2048, 4096, 8192, 16128]):
        cnt = 65536 if ell <= 8192 else 32768
        E = synth.exponent(ell, 0x5EEDC004)
        xs = synth.messages(n, cnt, 0x5EEDC004, 64)
        x = torch.from_numpy(xs.view(np.int32)).cuda()
        y = torch.empty_like(x)
        t = timed(torch, lambda: ctx.modexp(x, y, E), reps=2)
        s = 16 if ell > 4096 else 64
        ok = bool(np.array_equal(y.cpu().numpy().view(np.uint32)[:s], orc.modexp_batch(xs[:s], E, n, threads=os.cpu_count())))
        emit({"config": "C4", "exponent_bits": ell, "messages": cnt, "k": ctx.k, "modexps_per_s": cnt / t,
              "imad_eq_frac": cnt * bench.sliding_window_mm(E) * 2 * per_mm(ctx.k) / t / peak(),
              "bit_exact_sample": ok, "sample": s})


def wide(torch, mr, orc, quick):
    import random
    for bits in (4096, 8192, 16128):
        rng = random.Random(bits)
        N = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
        limbs = (bits + 31) // 32
        ctx = mr.RnsContext(N, limbs)
        for ell in (17, bits):
            E = 65537 if ell == 17 else rng.getrandbits(bits) | (1 << (bits - 1))
            # tensor-core wide kernel: k = 129 / 257 128-message tile-jobs (2 / 1 per SM: 37,888 / 18,944 = one per
            # tile), k = 505 64-message tile-jobs (9,472 = one per SM)
            cnt = 65536 if bits == 4096 and ell == 17 else 37888 if bits == 4096 else 9472 if bits == 16128 else 18944
            xs = synth.messages(N, cnt, 0x5EEDC0DE, limbs)
            x = torch.from_numpy(xs.view(np.int32)).cuda()
            y = torch.empty_like(x)
            t = timed(torch, lambda: ctx.modexp(x, y, E), reps=2 if ell == 17 else 1)
            s = 8 if ell == 17 else 1
            ok = bool(np.array_equal(y.cpu().numpy().view(np.uint32)[:s], orc.modexp_batch(xs[:s], E, N, threads=s)))
            emit({"config": "W", "modulus_bits": bits, "exponent_bits": ell, "messages": cnt, "k": ctx.k,
                  "modexps_per_s": cnt / t, "imad_eq_frac": cnt * bench.sliding_window_mm(E) * 2 * per_mm(ctx.k) / t / peak(),
                  "bit_exact_sample": ok, "sample": s})


def rng(torch, mr, quick):
    from oracle import drbg
    streams, nb = 16384, 65536                      # 1 GiB per request (2^19 bits per stream, the maximum)
    g = mr.Drbg(bytes(range(32)), bytes(range(16)), b"bench", streams)
    out = torch.empty(streams * nb, dtype=torch.uint8, device="cuda")
    t = timed(torch, lambda: g.generate(out, nb), reps=3)
    host = out[: 4 * nb].cpu().numpy().tobytes()
    # the sampled streams continue from the same state sequence as the oracle's (warm-up + 3 timed requests)
    ok = True
    for s in range(2):
        d = drbg.HashDrbg(bytes(range(32)), bytes(range(16)), drbg.stream_pers(b"bench", s))
        for _ in range(4):
            want = d.generate(nb)
        ok &= host[s * nb:(s + 1) * nb] == want
    nblk = streams * nb // 2500
    blocks = out[: nblk * 2500].view(nblk, 2500)
    stats = torch.empty((nblk, 16), dtype=torch.int32, device="cuda")
    th = timed(torch, lambda: mr.fips_health(blocks, stats), reps=3)
    v = stats[:, 15].cpu().numpy()
    emit({"config": "RNG", "streams": streams, "bytes_per_request": nb, "generate_GB_per_s": streams * nb / t / 1e9,
          "health_GB_per_s": nblk * 2500 / th / 1e9, "health_blocks": nblk,
          "health_pass_fraction": float((v == 15).mean()), "bit_exact_sample": bool(ok), "sample": "2 streams x 64 KiB",
          "paper_context": "32-40 GB/s of seed bits on 2013 GPUs (P:121)"})


MR_WINDOW = int(os.environ.get("MR_BENCH_WINDOW", "5"))   # fixed window of the a^d ladder (public API at 1024 bits: 5)


def c5(torch, mr, orc, quick):
    cnt = 16384 if quick else 65536
    rounds = 5
    ns = synth.limbs32_batch(0x5EEDC005, synth.TAG_CAND, 0, cnt, 32)
    ns[:, 0] |= 1
    ns[:, 31] |= 0xC0000000
    nints = [int.from_bytes(r.tobytes(), "little") for r in ns]
    bases = np.zeros((cnt, rounds, 32), dtype=np.uint32)
    for i in range(cnt):
        for r, b in enumerate(synth.mr_bases(nints[i], rounds, 0x5EEDC005, i)):
            bases[i, r] = np.frombuffer(b.to_bytes(128, "little"), dtype=np.uint32)
    d_n = torch.from_numpy(ns.view(np.int32)).cuda()
    d_b = torch.from_numpy(bases.view(np.int32)).cuda()
    v = torch.zeros(cnt, dtype=torch.uint8, device="cuda")
    w = torch.zeros(cnt, dtype=torch.int16, device="cuda")
    L = mr.lib()
    L.mr_internal_miller_rabin.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    stream = torch.cuda.current_stream().cuda_stream
    res = {}
    for forced in (1, 0):
        def run():
            rc = L.mr_internal_miller_rabin(d_n.data_ptr(), 32, cnt, d_b.data_ptr(), rounds, 0, v.data_ptr(),
                                            w.data_ptr(), None, 0, stream, forced, MR_WINDOW)
            assert rc == 0
        t = timed(torch, run, reps=2)
        res[forced] = (t, v.cpu().numpy().copy(), w.cpu().numpy().copy())
    s = 512
    fp = orc.base_primes(66)
    ov, ow = [], []
    for i in range(s):
        a, b = orc.miller_rabin(nints[i], [int.from_bytes(bases[i, r].tobytes(), "little") for r in range(rounds)], fp)
        ov.append(a)
        ow.append(b)
    same = bool(np.array_equal(res[1][1], res[0][1]) and np.array_equal(res[1][2], res[0][2]))
    ok = bool(list(res[0][1][:s]) == ov and list(res[0][2][:s]) == ow)
    mm_round = 15 + ((32 * 32 + 3) // 4) * 5 + 2        # fixed window w = 4: table + 256 x (4 sq + 1 mul) + checks
    rounds_needed = int(np.sum(np.where(res[0][2] >= 0, res[0][2] + 1, rounds)))
    emit({"config": "C5", "candidates": cnt, "rounds": rounds, "forced_rounds_per_s": cnt * rounds / res[1][0],
          "early_exit_candidates_per_s": cnt / res[0][0], "rounds_needed": rounds_needed,
          "probably_prime": int(np.sum(res[0][1] == 1)),
          "forced_imad_eq_frac": cnt * rounds * mm_round * 2 * per_mm(33) / res[1][0] / peak(),
          "verdicts_equal_forced_vs_early_exit": same, "bit_exact_sample_vs_oracle": ok, "sample": s})


def kg(torch, mr, quick):
    """GPU RSA key generation: keys/s, e = 65537; rounds = 5 (FIPS 186-4 C.3 count
    for 1024-bit primes is 4-5) and 64 (the fixture recipe).  Sample: 4 keys checked for n = p q and
    e d = 1 mod phi on the host."""
    for bits, cnt, rounds in ([(1024, 1024, 5), (2048, 256, 5)] if quick else
                              [(1024, 4096, 5), (1024, 16384, 5), (2048, 1024, 5), (2048, 4096, 5), (2048, 4096, 64),
                               (3072, 1024, 5)]):
        full, half = bits // 32, bits // 64
        bufs = [torch.zeros((cnt, full if f in ("n", "d") else half), dtype=torch.int32, device="cuda")
                for f in ("n", "p", "q", "d", "dp", "dq", "qinv")]
        mr.mr_rsa_keygen_batch(8, bits, 65537, 1, rounds, *[b[:8] for b in bufs])     # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mr.mr_rsa_keygen_batch(cnt, bits, 65537, 0x5EEDC0DE, rounds, *bufs)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        h = [b.cpu().numpy().view(np.uint32) for b in bufs]
        ok = True
        for i in range(4):
            n, p, q, d = (int.from_bytes(h[j][i].tobytes(), "little") for j in (0, 1, 2, 3))
            ok &= n == p * q and 65537 * d % ((p - 1) * (q - 1)) == 1
        emit({"config": "KG", "bits": bits, "keys": cnt, "mr_rounds": rounds, "seconds": t, "keys_per_s": cnt / t,
              "sample_valid": bool(ok), "timing": "host wall clock around the synchronous call"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C3,C4,C5")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    import torch

    import oracle
    import paper_1305_3699_b200 as mr
    torch.cuda.set_device(0)
    for c in a.configs.split(","):
        t0 = time.time()
        if c == "C1":
            c1(torch, mr, oracle)
        elif c == "C3":
            c3(torch, mr, oracle, a.quick)
        elif c == "C4":
            c4(torch, mr, oracle, a.quick)
        elif c == "C5":
            c5(torch, mr, oracle, a.quick)
        elif c == "RNG":
            rng(torch, mr, a.quick)
        elif c == "W":
            wide(torch, mr, oracle, a.quick)
        elif c == "KG":
            kg(torch, mr, a.quick)
        print(f"# {c} done in {time.time() - t0:.1f} s", file=sys.stderr)


if __name__ == "__main__":
    main()
