"""bench.py — BASELINE.json's metric on B200: RSA-2048 modexps/s (CRT decryptions), bit-exact.

Default workload (BASELINE.json configs[1], "C2"): RSA-2048 batched CRT decryption, 65,536 messages
per GPU, committed oracle-generated key tests/golden/keys/rsa2048.json, ciphertexts from the
SplitMix64 recipe of synth/ (DESIGN.md §6).  One step = one mr_rsa_decrypt_batch over the batch:
two half-size RNS-Montgomery ladders (k = 33) in one launch + the CRT recombination launch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--count C]

N > 1 runs under torchrun (one rank per GPU): every rank decrypts its own 65,536 messages (global
indices rank*C + i): weak scaling, no data-path collective (the messages are independent, DESIGN.md
§7); timing is max over ranks via all_reduce(MAX).  `--impl reference` times the CPU oracle (the
reference arm of this tier) on the same workload on the host cores.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RSA-2048 modexps/sec (1/2/4/8 B200) and % of INT32 IMAD peak, bit-exact vs CPU"
UNIT = "modexps/s"
SEED = 0x5EEDC002
K_HALF = 33                      # channels per base for 1024-bit CRT halves
SM_COUNT = 148
IMAD_PER_CLK_SM = 64             # tools/n9_intpeak: IMAD 63.9/clk/SM, IMAD.WIDE 30/clk/SM -> max(64, 2*30)


def load_key(name="rsa2048"):
    with open(os.path.join(ROOT, "tests", "golden", "keys", name + ".json")) as f:
        k = json.load(f)
    return {f: (int(v, 16) if isinstance(v, str) and f not in ("seed", "recipe") else v) for f, v in k.items()}


def sliding_window_mm(E: int) -> int:
    """Montgomery multiplications of a best-window sliding-window exponentiation of exponent E
    (table 2^(w-1) incl. the squaring, l-1 squarings, one multiply per window) + entry + exit
    (SURVEY.md §8(d) numerator definition)."""
    bits = E.bit_length()
    best = None
    for w in range(1, 8):
        n, i, first = 0, bits - 1, True
        while i >= 0:
            if not (E >> i) & 1:
                n += 1
                i -= 1
                continue
            lo = max(i - w + 1, 0)
            while not (E >> lo) & 1:
                lo += 1
            if first:
                first = False
            else:
                n += (i - lo + 1) + 1
            i = lo - 1
        cost = (1 << (w - 1) if w > 1 else 0) + n
        best = cost if best is None else min(best, cost)
    return best + 2


def imad_eq_per_decrypt(key) -> int:
    """algorithmic IMAD-eq per RSA CRT decryption: 2 x sum_h mm(d_h) x (2k^2 + 8k + 4) (§8(d))."""
    per_mm = 2 * K_HALF * K_HALF + 8 * K_HALF + 4
    return 2 * (sliding_window_mm(key["dp"]) + sliding_window_mm(key["dq"])) * per_mm


def peak_imad_eq_per_s(sm_mhz: float) -> float:
    return IMAD_PER_CLK_SM * SM_COUNT * sm_mhz * 1e6


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ reference arm: the CPU oracle

def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    key = load_key()
    threads = os.cpu_count() or 1
    per_step = args.ref_sample
    cs = synth.messages(key["n"], per_step, SEED, 64, edge=synth.edge_values(key["n"], key["p"], key["q"]))
    for _ in range(args.warmup):
        oracle.crt_decrypt_batch(cs, key["p"], key["q"], key["dp"], key["dq"], key["qinv"], 32, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.crt_decrypt_batch(cs, key["p"], key["q"], key["dp"], key["dq"], key["qinv"], 32, threads)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": workload_config(args, reference=True),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{per_step} RSA-2048 CRT decryptions per step (oracle/oracle.c, "
                                       f"{threads} pthreads)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, reference=False):
    return {"workload": "C2: RSA-2048 batched CRT decryption, 65,536 messages per GPU (BASELINE configs[1])",
            "key": "tests/golden/keys/rsa2048.json (oracle-generated, seed 0x5EEDC002)",
            "messages_per_gpu": args.count, "rns_k_per_half": K_HALF, "modulus_bits": 2048,
            "base_extension": "imad" if os.environ.get("MR_RNS_IMAD_ONLY", "0") == "1" else "tcgen05-i8",
            "inputs": "SplitMix64 ciphertexts uniform in [0, N) + edge values (synth/)",
            "l2": "flushed between timed steps (256 MiB write)" if not reference else "n/a (CPU)"}


# ------------------------------------------------------------------ our arm

def run_ours(args, world, rank, local):
    import torch

    import paper_1305_3699_b200 as mr
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    key = load_key()
    count = args.count
    first = rank * count
    cs = synth.messages(key["n"], count, SEED, 64, edge=synth.edge_values(key["n"], key["p"], key["q"]), first=first)
    priv = mr.RsaPrivateKey(key["p"], key["q"], key["dp"], key["dq"], key["qinv"], device=local)
    c = torch.from_numpy(cs.view(np.int32)).to(dev)
    m = torch.empty_like(c)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)   # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    L = mr.lib()
    import ctypes
    L.mr_internal_timing.argtypes = [ctypes.c_int]

    # warm-up (untimed)
    for _ in range(args.warmup):
        priv.decrypt(c, m)
    torch.cuda.synchronize()

    # correctness spot check of the benchmarked launch against the oracle (outside the timed region)
    verified = None
    if rank == 0 and not args.no_verify:
        import oracle
        idx = list(range(0, 64)) + list(range(64, count, max(1, count // 192)))
        ref = oracle.crt_decrypt_batch(cs[idx], key["p"], key["q"], key["dp"], key["dq"], key["qinv"], 32,
                                       os.cpu_count() or 1)
        got = m.cpu().numpy().view(np.uint32)[idx]
        verified = {"sampled": len(idx), "mismatches": int((got != ref).any(axis=1).sum())}

    # timed region: K steps, each bracketed by CUDA events on the launching stream; L2 flushed between
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    L.mr_internal_timing(1)
    L.mr_internal_timing_collect(None, None, None, None)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i)
            ev[i][0].record(stream)
            priv.decrypt(c, m)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    L.mr_internal_timing(0)
    ms_l, n_l, ms_c, n_c = ctypes.c_double(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
    L.mr_internal_timing_collect(ctypes.byref(ms_l), ctypes.byref(n_l), ctypes.byref(ms_c), ctypes.byref(n_c))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    total_ms_max = max_over_ranks(total_ms, world, dev)
    value = count * world * args.steps / (total_ms_max / 1e3)

    # end-to-end through the public API with pinned host buffers: every step copies its ciphertexts
    # host->device, decrypts and copies its plaintexts device->host.  Double-buffered on three streams
    # (H2D, compute, D2H), so step i+1's upload and step i-1's download overlap step i's decryption.
    h_c = torch.from_numpy(cs.view(np.int32)).pin_memory()
    h_m = [torch.empty_like(h_c).pin_memory() for _ in range(2)]
    d_c = [torch.empty_like(c) for _ in range(2)]
    d_m = [torch.empty_like(c) for _ in range(2)]
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    up_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    dn_done = [torch.cuda.Event() for _ in range(2)]

    def e2e_steps(n):
        for i in range(n):
            b = i % 2
            s_up.wait_event(comp_done[b])                 # d_c[b] no longer read by step i-2
            with torch.cuda.stream(s_up):
                d_c[b].copy_(h_c, non_blocking=True)
            up_done[b].record(s_up)
            stream.wait_event(up_done[b])
            stream.wait_event(dn_done[b])                 # d_m[b] downloaded by step i-2
            priv.decrypt(d_c[b], d_m[b])
            comp_done[b].record(stream)
            s_dn.wait_event(comp_done[b])
            with torch.cuda.stream(s_dn):
                h_m[b].copy_(d_m[b], non_blocking=True)
            dn_done[b].record(s_dn)
        stream.wait_event(dn_done[(n - 1) % 2])
        stream.wait_event(dn_done[n % 2])

    for ev_ in comp_done + dn_done:
        ev_.record(stream)
    e2e_steps(2)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s_up.wait_event(e0)
    e2e_steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world, dev)
    e2e_value = count * world * args.steps / (e2e_ms / 1e3)
    ref_m = m.cpu().numpy()
    e2e_ok = bool(all(np.array_equal(h.numpy(), ref_m) for h in h_m))

    # roofline of the dominant kernel (the ladder launch): algorithmic IMAD-eq / its event time
    clocks = clk.summary()
    per_dec = imad_eq_per_decrypt(key)
    ladder_ms = ms_l.value / max(1, n_l.value)
    achieved = per_dec * count / (ladder_ms / 1e3)                   # IMAD-eq/s per GPU
    peak = peak_imad_eq_per_s(measured_peaks().get("sm_max_mhz", 1965.0))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(key)
    if rank != 0:
        return
    tensor = os.environ.get("MR_RNS_IMAD_ONLY", "0") != "1"
    kname = "k_modexp_tc (CRT half-ladders, k=33, base extensions on tcgen05 int8)" if tensor else \
        "k_modexp (CRT half-ladders, k=33, IMAD-pipe base extensions)"
    # tensor-core work of the two base extensions: useful u8 MACs per Montgomery multiplication
    # = 2 x (4k)^2, 2 ops each; peak = measured bf16 burst x (4.5 / 2.25) nominal i8:bf16 ratio
    mm_per_dec = 2 * (sliding_window_mm(key["dp"]) + sliding_window_mm(key["dq"])) // 2
    i8_ops_per_dec = 2 * mm_per_dec * 2 * (4 * K_HALF) ** 2 if tensor else 0
    i8_peak = measured_peaks().get("bf16_tflops", 1611.6) * 2.0 * 1e12
    i8_achieved = i8_ops_per_dec * count / (ladder_ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic", "config": workload_config(args),
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12,
                     "unit": "T IMAD-eq/s (INT32 IMAD pipe, 64/clk/SM x 148 SM x 1965 MHz)",
                     "frac": achieved / peak, "traffic": ncu_traffic(tensor, count),
                     "kernel": kname, "ladder_ms_per_launch": ladder_ms,
                     "tensor_i8": {"achieved_tops": i8_achieved / 1e12, "peak_tops": i8_peak / 1e12,
                                   "frac": i8_achieved / i8_peak,
                                   "peak_source": "MEASURED_PEAKS bf16_tflops x 2 (nominal i8:bf16 4.5:2.25)"}
                     if tensor else None,
                     "cuda_core_pipes_ncu": ncu_pipes(tensor, count),
                     "combine_ms_per_launch": ms_c.value / max(1, n_c.value),
                     "imad_eq_per_decrypt": per_dec,
                     "frac_at_median_clock": (achieved / peak_imad_eq_per_s(clocks["sm_mhz"]))
                     if clocks.get("sm_mhz") else None},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(cs.nbytes),
                "d2h_bytes_per_step": int(cs.nbytes), "bit_identical_to_device_run": e2e_ok,
                "transfers": "pinned host buffers, double-buffered: H2D / decrypt / D2H streams overlap across steps"},
        "gpu_launches": n_l.value + n_c.value,
        "clocks": clocks,
        "verified": verified,
    }
    print(json.dumps(line), flush=True)


def ncu_record(tensor: bool, count: int):
    """the committed ncu --set full summary of the ladder kernel in this configuration
    (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{'k_modexp_tc' if tensor else 'k_modexp'}/c2/{count}")
    except (OSError, ValueError):
        return None


def ncu_traffic(tensor: bool, count: int):
    """DRAM bytes (read + write) per launch of the ladder kernel from the committed ncu capture."""
    rec = ncu_record(tensor, count)
    return None if rec is None else rec["dram_bytes_read"] + rec["dram_bytes_write"]


def ncu_pipes(tensor: bool, count: int):
    """utilisation of the binding CUDA-core resources from the same capture (issue slots, FMA-heavy pipe)."""
    rec = ncu_record(tensor, count)
    if rec is None or "issue_active_pct" not in rec:
        return None
    return {k: rec[k] for k in ("issue_active_pct", "fmaheavy_pipe_pct", "alu_pipe_pct", "tensor_imma_pct",
                                "warp_instructions_per_multiplication", "source") if k in rec}


def cpu_baseline(key, budget_s: float = 10.0):
    """the oracle, as it stands, on the host cores: a bounded sample of the same workload."""
    import oracle
    threads = os.cpu_count() or 1
    n = 64 * threads
    cs = synth.messages(key["n"], n, SEED, 64)
    t0 = time.perf_counter()
    done = 0
    while True:
        oracle.crt_decrypt_batch(cs, key["p"], key["q"], key["dp"], key["dq"], key["qinv"], 32, threads)
        done += n
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{done} RSA-2048 CRT decryptions of the C2 workload in {dt:.1f} s "
                      f"(oracle/oracle.c, {threads} pthreads)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--count", type=int, default=65536, help="messages per GPU")
    ap.add_argument("--ref-sample", type=int, default=512, help="reference arm: decryptions per step")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
