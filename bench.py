"""bench.py — BASELINE.json's metric on B200: RSA-2048 modexps/s (CRT decryptions), bit-exact.

Default workload (BASELINE.json configs[1], "C2"): RSA-2048 batched CRT decryption, 65,536 messages
per GPU, committed oracle-generated key tests/golden/keys/rsa2048.json, ciphertexts from the
SplitMix64 recipe of synth/ (DESIGN.md §6).  One step = one mr_rsa_decrypt_batch over the batch:
two half-size RNS-Montgomery ladders (k = 33) in one launch + the CRT recombination launch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3dec|c3enc|c5] [--count C | --total T] [--dry-run-cpu]

Multi-GPU: one process per GPU.  `--gpus N` with N > 1 outside torchrun re-launches
itself under `torch.distributed.run` (127.0.0.1).  Units are independent, so the data path has no
collective: rank r owns the contiguous global indices [r*n/N, (r+1)*n/N) — `--count C` per GPU (weak
scaling, the default) or `--total T` split over the ranks (strong scaling, the C3 1K-1M sweep).  The
timed device region is max over ranks (all_reduce MAX of CUDA-event times).  The end-to-end region adds,
every step, the pinned H2D copy of the rank's inputs, the final gather (all_gather_into_tensor of the
outputs; Miller-Rabin: verdicts and witness rounds) and rank 0's D2H read of the gathered result.  After
it, rank 0 checks the gathered bytes against the oracle on a sample of global indices and, for N > 1,
byte-for-byte against a single-GPU run of the whole batch on its own device (the G = 1 identity, T6).

`--impl reference` times the CPU oracle (this tier's reference arm) on a bounded sample of the same
workload on the host cores.  `--dry-run-cpu` exercises the multi-rank host path (sharding, gloo gather,
identity check) on a CPU-only box with the oracle standing in for the device call: it prints a line
marked `"dry_run": true` with no throughput and is never a measurement.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
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
IMAD_PER_CLK_SM = 64             # profiles/r2_peaks_int.json (tools/n9_intpeak): max(IMAD, 2 x IMAD.WIDE) per clk/SM


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


def per_mm(k: int) -> int:
    """algorithmic word products of one RNS Montgomery multiplication: 2k^2 + 8k + 4."""
    return 2 * k * k + 8 * k + 4


def imad_eq_per_decrypt(key) -> int:
    """algorithmic IMAD-eq per RSA CRT decryption: 2 x sum_h mm(d_h) x (2k^2 + 8k + 4) (§8(d))."""
    return 2 * (sliding_window_mm(key["dp"]) + sliding_window_mm(key["dq"])) * per_mm(K_HALF)


def mr_round_mm(bits: int = 1024, w: int = 5) -> int:
    """Montgomery multiplications of one forced Miller-Rabin round over `bits`-bit candidates with the
    fixed-window a^d ladder (R6): 2^(w-1)+1 table entries, bits squarings, bits/w window
    multiplies, entry and exit (the s-1 squarings of the round's tail are < 1 % and not counted)."""
    return (1 << (w - 1)) + 1 + bits + (bits + w - 1) // w + 2


def peak_imad_eq_per_s(sm_mhz: float) -> float:
    return IMAD_PER_CLK_SM * SM_COUNT * sm_mhz * 1e6


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def i8_peak():
    """(ops/s, source) of the int8 tensor cores: profiles/r2_tc_i8_peak.jsonl (tools/tc_i8_peak.cu, the
    largest single-CTA MMA, M=128 N=256, back to back, all SMs), else MEASURED_PEAKS bf16 x 2 (nominal)."""
    path = os.path.join(ROOT, "profiles", "r2_tc_i8_peak.jsonl")
    try:
        best = 0.0
        with open(path) as f:
            for line in f:
                r = json.loads(line)
                if "tops" in r and "N=256" in r.get("shape", "") and "cta_group::1" in r["shape"]:
                    best = max(best, r["tops"])
        if best > 0:
            return best * 1e12, "profiles/r2_tc_i8_peak.jsonl (tcgen05.mma kind::i8 M=128 N=256 K=32, 148 SMs, measured)"
    except (OSError, ValueError):
        pass
    return measured_peaks().get("bf16_tflops", 1631.6) * 2.0 * 1e12, "MEASURED_PEAKS bf16_tflops x 2 (nominal i8:bf16)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index = index
        self.proc = None
        self.enabled = enabled

    def __enter__(self):
        if not self.enabled:
            return self
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


# ------------------------------------------------------------------ process groups

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: run N ranks of this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "gloo" if (args.impl == "reference" or args.dry_run_cpu) else "nccl"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        if not dist.is_initialized():
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


def shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """contiguous global-index range [lo, hi) of rank `rank`: the first n_total % world
    ranks take one more unit."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


# ------------------------------------------------------------------ workloads

class Workload:
    """One BASELINE configuration: seeded inputs by global index, the library call of one step, the
    oracle on a sample, and the algorithmic work per unit."""

    name = ""
    describe = ""
    unit = UNIT
    metric = METRIC

    def inputs(self, lo: int, hi: int) -> list[np.ndarray]:
        raise NotImplementedError

    def out_shapes(self, n: int) -> list[tuple]:
        raise NotImplementedError

    def oracle(self, ins: list[np.ndarray], threads: int) -> list[np.ndarray]:
        raise NotImplementedError


class CrtDecrypt(Workload):
    def __init__(self, key_name: str, seed: int, k: int, describe: str):
        self.key = load_key(key_name)
        self.seed, self.k = seed, k
        self.L = self.key["bits"] // 32 if "bits" in self.key else (self.key["n"].bit_length() + 31) // 32
        self.describe = describe
        self.mm = sliding_window_mm(self.key["dp"]) + sliding_window_mm(self.key["dq"])

    def inputs(self, lo, hi):
        k = self.key
        return [synth.messages(k["n"], hi - lo, self.seed, self.L, edge=synth.edge_values(k["n"], k["p"], k["q"]),
                               first=lo)]

    def out_shapes(self, n):
        return [((n, self.L), "int32")]

    def make_device_step(self, mr, device):
        k = self.key
        priv = mr.RsaPrivateKey(k["p"], k["q"], k["dp"], k["dq"], k["qinv"], device=device)
        self._keep = priv
        return lambda ins, outs: priv.decrypt(ins[0], outs[0])

    def oracle(self, ins, threads):
        import oracle
        k = self.key
        return [oracle.crt_decrypt_batch(ins[0], k["p"], k["q"], k["dp"], k["dq"], k["qinv"], self.L // 2, threads)]

    def work(self):
        """(tensor-core ops, CUDA-core elementwise IMAD-eq, all-work IMAD-eq) per unit"""
        k = self.k
        tensor = 2 * 16 * 2 * k * (k + 1) * self.mm          # 2 ops per u8 MAC, 16 u8 MACs per word product
        elementwise = 2 * (6 * k + 4) * self.mm
        return tensor, elementwise, 2 * per_mm(k) * self.mm


class Encrypt(Workload):
    def __init__(self, key_name: str, seed: int, describe: str):
        self.key = load_key(key_name)
        self.seed = seed
        self.L = (self.key["n"].bit_length() + 31) // 32
        self.describe = describe
        self.k = None
        self.mm = sliding_window_mm(self.key["e"])

    def inputs(self, lo, hi):
        k = self.key
        return [synth.messages(k["n"], hi - lo, self.seed, self.L, edge=synth.edge_values(k["n"], k["p"], k["q"]),
                               first=lo)]

    def out_shapes(self, n):
        return [((n, self.L), "int32")]

    def make_device_step(self, mr, device):
        ctx = mr.RnsContext(self.key["n"], self.L, device=device)
        self.k = ctx.k
        self._keep = ctx
        return lambda ins, outs: ctx.encrypt(ins[0], outs[0], self.key["e"])

    def oracle(self, ins, threads):
        import oracle
        return [oracle.modexp_batch(ins[0], self.key["e"], self.key["n"], threads)]

    def work(self):
        k = self.k or (self.key["n"].bit_length() // 32 + 1)
        # k = 97 / 129 run on the tensor-core wide kernel (base extensions on tcgen05) unless it is switched off
        tensor = 2 * 16 * 2 * k * (k + 1) * self.mm if tcw_enabled() else 0
        elementwise = 2 * (6 * k + 4) * self.mm if tcw_enabled() else 2 * per_mm(k) * self.mm
        return tensor, elementwise, 2 * per_mm(k) * self.mm


class MillerRabin(Workload):
    """C5: forced Miller-Rabin rounds (every round for every candidate) on seeded 1024-bit candidates that
    survive nothing in particular (uniform odd, top two bits set), R = 5 bases each (tag BASE)."""

    unit = "MR rounds/s"
    metric = "RSA-2048 key generation: Miller-Rabin rounds/s on 1024-bit candidates (1/2/4/8 B200), bit-exact vs CPU"

    def __init__(self, rounds=5, seed=0x5EEDC005):
        self.R, self.seed, self.L, self.k = rounds, seed, 32, 33
        self.describe = f"C5: Miller-Rabin, {rounds} forced rounds per seeded 1024-bit candidate (BASELINE configs[4])"

    def inputs(self, lo, hi):
        ns = synth.limbs32_batch(self.seed, synth.TAG_CAND, lo, hi - lo, self.L)
        ns[:, 0] |= 1
        ns[:, self.L - 1] |= 0xC0000000
        bases = np.zeros((hi - lo, self.R, self.L), dtype=np.uint32)
        for i in range(hi - lo):
            n = int.from_bytes(ns[i].tobytes(), "little")
            for r, b in enumerate(synth.mr_bases(n, self.R, self.seed, lo + i)):
                bases[i, r] = np.frombuffer(b.to_bytes(4 * self.L, "little"), dtype=np.uint32)
        return [ns, bases.reshape(hi - lo, self.R * self.L)]

    def out_shapes(self, n):
        return [((n,), "uint8"), ((n,), "int16")]

    def make_device_step(self, mr, device):
        import ctypes

        import torch
        L = mr.lib()
        L.mr_internal_miller_rabin.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                               ctypes.c_int]

        def step(ins, outs):
            n = ins[0].shape[0]
            rc = L.mr_internal_miller_rabin(ins[0].data_ptr(), self.L, n, ins[1].data_ptr(), self.R, 0,
                                            outs[0].data_ptr(), outs[1].data_ptr(), None, device,
                                            torch.cuda.current_stream().cuda_stream, 1, 5)
            if rc:
                raise RuntimeError(f"mr_internal_miller_rabin failed: {rc}")
        return step

    def oracle(self, ins, threads):
        import oracle
        fp = oracle.base_primes(2 * self.k)
        v, w = oracle.miller_rabin_batch(ins[0], ins[1].reshape(-1, self.R, self.L), fp, threads)
        return [v.astype(np.uint8), w.astype(np.int16)]

    def units(self, n):
        return n * self.R

    def work(self):
        mm = mr_round_mm(32 * self.L, 5)
        k = self.k
        return 2 * 16 * 2 * k * (k + 1) * mm, 2 * (6 * k + 4) * mm, 2 * per_mm(k) * mm


def make_workload(name: str) -> Workload:
    if name == "c2":
        return CrtDecrypt("rsa2048", SEED, K_HALF,
                          "C2: RSA-2048 batched CRT decryption (BASELINE configs[1])")
    if name == "c3dec":
        return CrtDecrypt("rsa3072", 0x5EEDC003, 49, "C3: RSA-3072 batched CRT decryption (BASELINE configs[2])")
    if name == "c3enc":
        return Encrypt("rsa3072", 0x5EEDC003, "C3: RSA-3072 batched encryption, e = 65537 (BASELINE configs[2])")
    if name == "c5":
        return MillerRabin()
    raise SystemExit(f"unknown workload {name}")


def units_of(wl: Workload, n: int) -> int:
    return wl.units(n) if hasattr(wl, "units") else n


# ------------------------------------------------------------------ devices: the B200, or the CPU dry run

class CudaDevice:
    dry = False

    def __init__(self, local: int):
        import torch
        self.torch = torch
        if not torch.cuda.is_available():
            raise SystemExit("bench.py: no CUDA device (there is no CPU fallback; --dry-run-cpu only exercises the "
                             "multi-rank host path with the oracle standing in for the device)")
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.index = local
        self.stream = torch.cuda.current_stream(self.dev)

    def put(self, a: np.ndarray):
        return self.torch.from_numpy(_as_signed(a)).to(self.dev)

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=getattr(self.torch, dtype), device=self.dev)

    def host(self, t) -> np.ndarray:
        return t.cpu().numpy()

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def sync(self):
        self.torch.cuda.synchronize()


def _as_signed(a: np.ndarray) -> np.ndarray:
    return a.view(np.int32) if a.dtype == np.uint32 else a


class CpuDryRun:
    """the device call replaced by the oracle on CPU tensors (gloo); host-path coverage only."""

    dry = True

    def __init__(self, wl: Workload):
        import torch
        self.torch = torch
        self.dev = torch.device("cpu")
        self.index = 0
        self.stream = None
        self.wl = wl

    def put(self, a):
        return self.torch.from_numpy(_as_signed(np.ascontiguousarray(a)).copy())

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=getattr(self.torch, dtype))

    def host(self, t):
        return t.numpy()

    def event(self):
        class _Ev:
            def record(self, *a):
                self.t = time.perf_counter()

            def elapsed_time(self, other):
                return (other.t - self.t) * 1e3
        return _Ev()

    def sync(self):
        pass

    def step_fn(self):
        def step(ins, outs):
            res = self.wl.oracle([_unsigned(i.numpy()) for i in ins], 1)
            for o, r in zip(outs, res):
                o.copy_(self.torch.from_numpy(_as_signed(np.ascontiguousarray(r)).reshape(o.shape)))
        return step


def _unsigned(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint32) if a.dtype == np.int32 else a


# ------------------------------------------------------------------ reference arm: the CPU oracle

def run_reference(args, world, rank):
    if rank != 0:
        return
    wl = make_workload(args.workload)
    threads = os.cpu_count() or 1
    per_step = args.ref_sample
    ins = wl.inputs(0, per_step)
    for _ in range(args.warmup):
        wl.oracle(ins, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.oracle(ins, threads)
    dt = time.perf_counter() - t0
    value = units_of(wl, per_step) * args.steps / dt
    cfg = {"workload": wl.describe, "sample_per_step": per_step,
           "note": f"the oracle (oracle/oracle.c, plain positional bignums) on {per_step} units of the same "
                   f"seeded workload per step, {threads} host threads; not the GPU batch size",
           "inputs": "SplitMix64 inputs by global index (synth/), the first units of the GPU batch"}
    line = {"metric": wl.metric, "value": value, "unit": wl.unit, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": wl.unit, "cores": threads, "cpu_model": cpu_model(),
                             "kind": "oracle",
                             "sample": f"{per_step} units per step x {args.steps} steps (oracle/oracle.c, "
                                       f"{threads} pthreads)"},
            "e2e": {"value": value, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def run_rank(args, world, rank, dev, wl: Workload, step):
    """The per-rank body of a bench run (shared by the B200 path and the CPU dry run).  Returns the JSON
    line on rank 0, None elsewhere."""
    torch = dev.torch
    import torch.distributed as dist
    total = args.total if args.total else args.count * world
    lo, hi = shard(total, world, rank)
    n_loc = hi - lo
    rows = -(-total // world)                               # gather rows per rank (padded to equal shards)
    ins_h = wl.inputs(lo, hi)
    ins = [dev.put(a) for a in ins_h]
    outs = [dev.empty(s, d) for s, d in wl.out_shapes(n_loc)]
    flush = None if dev.dry else dev.empty((64 * 1024 * 1024,), "int32")      # 256 MiB > 126 MB L2

    for _ in range(args.warmup):
        step(ins, outs)
    dev.sync()

    # ---- timed region: K steps, CUDA events on the launching stream; L2 flushed between steps
    lib = None
    if not dev.dry:
        import ctypes

        import paper_1305_3699_b200 as mr
        lib = mr.lib()
        lib.mr_internal_timing.argtypes = [ctypes.c_int]
        lib.mr_internal_timing(1)
        lib.mr_internal_timing_collect(None, None, None, None)
    ev = [(dev.event(), dev.event()) for _ in range(args.steps)]
    barrier(world)
    dev.sync()
    with ClockSampler(dev.index, enabled=not dev.dry) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i)
            ev[i][0].record(dev.stream) if dev.stream is not None else ev[i][0].record()
            step(ins, outs)
            ev[i][1].record(dev.stream) if dev.stream is not None else ev[i][1].record()
        dev.sync()
    barrier(world)
    launch = None
    if lib is not None:
        import ctypes
        lib.mr_internal_timing(0)
        ms_l, n_l, ms_c, n_c = ctypes.c_double(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        lib.mr_internal_timing_collect(ctypes.byref(ms_l), ctypes.byref(n_l), ctypes.byref(ms_c), ctypes.byref(n_c))
        ms_m, n_m = ctypes.c_double(), ctypes.c_int()
        lib.mr_internal_timing_mr(ctypes.byref(ms_m), ctypes.byref(n_m))
        if n_m.value:   # Miller-Rabin: each timed call is k_mr_setup + k_mr_rounds_tc (the ladder-kind slot)
            launch = (ms_m.value, n_m.value, 0.0, n_m.value)
        else:
            launch = (ms_l.value, n_l.value, ms_c.value, n_c.value)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    total_ms_max = max_over_ranks(total_ms, world, dev.dev if not dev.dry else None)
    value = units_of(wl, total) * args.steps / (total_ms_max / 1e3)

    # ---- end to end through the public API: pinned H2D of this rank's inputs, the step, the final gather
    # (all_gather_into_tensor over NCCL / NVLink), rank 0's D2H of the gathered outputs; double-buffered on
    # three streams so step i+1's upload and step i-1's download overlap step i.
    pin = (lambda t: t) if dev.dry else (lambda t: t.pin_memory())
    h_in = [pin(torch.from_numpy(_as_signed(np.ascontiguousarray(a)))) for a in ins_h]
    gshapes = [((rows * world,) + tuple(s[1:]), d) for s, d in wl.out_shapes(rows)]
    d_in = [[dev.empty(tuple(a.shape), str(a.dtype).replace("torch.", "")) for a in h_in] for _ in range(2)]
    d_out = [[dev.empty(((rows,) + tuple(s[1:])), d) for s, d in wl.out_shapes(rows)] for _ in range(2)]
    d_all = [[dev.empty(s, d) for s, d in gshapes] for _ in range(2)]
    h_all = [[pin(torch.empty(s, dtype=getattr(torch, d))) for s, d in gshapes] for _ in range(2)]
    if not dev.dry:
        for b in range(2):
            for o in d_out[b]:
                o.zero_()                                     # padding rows of a short shard gather as zeros

    def gather(src, dst):
        if world == 1:
            dst.copy_(src)
        elif src.dtype in (torch.int16,):                     # NCCL has no int16: gather the bytes
            dist.all_gather_into_tensor(dst.view(torch.uint8), src.view(torch.uint8))
        else:
            dist.all_gather_into_tensor(dst, src)

    if dev.dry:
        def e2e_steps(n):
            for i in range(n):
                b = i % 2
                for d, h in zip(d_in[b], h_in):
                    d.copy_(h)
                step(d_in[b], [o[:n_loc] for o in d_out[b]])
                for o, a in zip(d_out[b], d_all[b]):
                    gather(o, a)
                if rank == 0:
                    for a, h in zip(d_all[b], h_all[b]):
                        h.copy_(a)
        e2e_steps(2)
        barrier(world)
        t0 = time.perf_counter()
        e2e_steps(args.steps)
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
        last = (args.steps - 1) % 2
    else:
        stream = dev.stream
        s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
        up_done = [torch.cuda.Event() for _ in range(2)]
        comp_done = [torch.cuda.Event() for _ in range(2)]
        dn_done = [torch.cuda.Event() for _ in range(2)]

        def e2e_steps(n):
            for i in range(n):
                b = i % 2
                s_up.wait_event(comp_done[b])                  # d_in[b] no longer read by step i-2
                with torch.cuda.stream(s_up):
                    for d, h in zip(d_in[b], h_in):
                        d.copy_(h, non_blocking=True)
                up_done[b].record(s_up)
                stream.wait_event(up_done[b])
                stream.wait_event(dn_done[b])                  # d_all[b] downloaded by step i-2
                step(d_in[b], [o[:n_loc] for o in d_out[b]])
                for o, a in zip(d_out[b], d_all[b]):           # the final gather, on the compute stream
                    gather(o, a)
                comp_done[b].record(stream)
                s_dn.wait_event(comp_done[b])
                if rank == 0:
                    with torch.cuda.stream(s_dn):
                        for a, h in zip(d_all[b], h_all[b]):
                            h.copy_(a, non_blocking=True)
                dn_done[b].record(s_dn)
            stream.wait_event(dn_done[(n - 1) % 2])
            stream.wait_event(dn_done[n % 2])

        for e in comp_done + dn_done:
            e.record(stream)
        e2e_steps(2)
        dev.sync()
        barrier(world)
        e0, e1 = dev.event(), dev.event()
        e0.record(stream)
        s_up.wait_event(e0)
        e2e_steps(args.steps)
        e1.record(stream)
        dev.sync()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1), world, dev.dev)
        last = (args.steps - 1) % 2
    e2e_value = units_of(wl, total) * args.steps / (e2e_ms / 1e3)

    # ---- G = 1 identity: rank 0 runs the WHOLE batch alone on its device and compares bytes
    identity = None
    if world > 1 and rank == 0 and not args.no_identity:
        full_in = [dev.put(a) for a in wl.inputs(0, total)]
        full_out = [dev.empty(s, d) for s, d in wl.out_shapes(total)]
        step(full_in, full_out)
        dev.sync()
        eq = True
        for a, f in zip(h_all[last], full_out):
            g = a.numpy().reshape(world, rows, *a.shape[1:])
            parts = [g[r, :shard(total, world, r)[1] - shard(total, world, r)[0]] for r in range(world)]
            eq &= bool(np.array_equal(np.concatenate(parts), dev.host(f)))
        identity = {"gathered_equals_single_gpu_run": eq, "units": total}
        del full_in, full_out
    barrier(world)
    if rank != 0:
        return None

    # ---- oracle sample of the gathered result (global indices)
    verified = None
    if not args.no_verify:
        idx = sorted(set(list(range(min(total, 64))) + list(range(64, total, max(1, total // 192)))))
        g = [a.numpy().reshape(world, rows, *a.shape[1:]) for a in h_all[last]]
        got = []
        for gi in g:
            parts = [gi[r, :shard(total, world, r)[1] - shard(total, world, r)[0]] for r in range(world)]
            got.append(np.concatenate(parts)[idx])
        ins_s = [np.concatenate([wl.inputs(i, i + 1)[j] for i in idx]) for j in range(len(ins_h))]
        ref = wl.oracle(ins_s, os.cpu_count() or 1)
        mism = sum(int((_unsigned(np.asarray(a)).reshape(len(idx), -1) != np.asarray(r).reshape(len(idx), -1)
                        ).any(axis=1).sum()) for a, r in zip(got, ref))
        verified = {"sampled": len(idx), "mismatches": mism, "of": "the gathered outputs (global indices) vs oracle"}

    line = {"metric": wl.metric, "value": None if dev.dry else value, "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.total else "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic", "config": workload_config(args, wl, total, world),
            "e2e": {"value": None if dev.dry else e2e_value, "unit": wl.unit,
                    "h2d_bytes_per_step": int(sum(a.nbytes for a in ins_h)),
                    "d2h_bytes_per_step": int(sum(h.numel() * h.element_size() for h in h_all[last])),
                    "gather": "all_gather_into_tensor of every rank's outputs per step" if world > 1 else
                              "single GPU: outputs copied as-is",
                    "transfers": "pinned host buffers, double-buffered: H2D / step + gather / D2H streams overlap"},
            "verified": verified, "identity_vs_single_gpu": identity}
    if dev.dry:
        line.update({"dry_run": True, "impl": "cpu-dry-run: the oracle stands in for the device call; NOT a "
                                              "measurement (host-path coverage: sharding, gloo gather, identity)"})
        return line
    clocks = clk.summary()
    line["clocks"] = clocks
    line["gpu_launches"] = (launch[1] + launch[3]) if launch else None
    line["roofline"] = roofline(wl, n_loc, launch, clocks, world, total_ms / args.steps)
    if not args.no_cpu_baseline and (world == 1 or args.cpu_baseline_multi):
        line["cpu_baseline"] = cpu_baseline(wl)
    return line


def roofline(wl: Workload, n_loc: int, launch, clocks, world, step_ms: float):
    """the dominant kernel (the ladder launch) against its binding roofline.  Work per unit is algorithmic
    (SURVEY §8(d)): tensor ops = 2 x 16 u8 MACs x 2k(k+1) base-extension word products per Montgomery
    multiplication; CUDA-core IMAD-eq = 2 x (6k + 4) elementwise word products per multiplication.  The
    roofline time is the larger of (tensor ops / i8 tensor peak) and (IMAD-eq / INT32 IMAD peak); `frac`
    is that pipe's achieved / peak.  The all-work IMAD-eq rate over the IMAD peak (what an IMAD-only
    implementation could reach at most) is reported separately as imad_eq_speedup."""
    ms_l, n_l, ms_c, n_c = launch
    # ladder (or Miller-Rabin) launches are timed by the library hook on their own stream
    ladder_ms = ms_l / n_l if n_l else step_ms
    t_ops, e_ops, all_ops = wl.work()
    units = units_of(wl, n_loc)
    sec = ladder_ms / 1e3
    imad_peak = peak_imad_eq_per_s(measured_peaks().get("sm_max_mhz", 1965.0))
    tpk, tsrc = i8_peak()
    t_ach = t_ops * units / sec
    e_ach = e_ops * units / sec
    t_time, e_time = t_ops / tpk, e_ops / imad_peak
    if t_ops and t_time >= e_time:
        bound, ach, pk, unit, fr = "tensor", t_ach / 1e12, tpk / 1e12, "TOPS (u8 x u8 MAC = 2 ops)", t_ach / tpk
    else:
        bound, ach, pk, unit, fr = "alu", e_ach / 1e12, imad_peak / 1e12, "T IMAD-eq/s (INT32 IMAD pipe)", e_ach / imad_peak
    rec = ncu_record(wl.name, n_loc)
    return {"bound": bound, "achieved": ach, "peak": pk, "unit": unit, "frac": fr,
            "traffic": None if rec is None else rec["dram_bytes_read"] + rec["dram_bytes_write"],
            "kernel": kernel_name(wl), "ladder_ms_per_launch": ladder_ms,
            "combine_ms_per_launch": ms_c / max(1, n_c) if n_c and ms_c else None,
            "peak_source": tsrc if bound == "tensor" else
            "64 IMAD-eq/clk/SM x 148 SM x sm_max_mhz (profiles/r2_peaks_int.json: IMAD 64/clk/SM, IMAD.WIDE 32)",
            "tensor_i8": {"achieved_tops": t_ach / 1e12, "peak_tops": tpk / 1e12, "frac": t_ach / tpk,
                          "source": tsrc} if t_ops else None,
            "cuda_core_elementwise": {"achieved_t_imad_eq": e_ach / 1e12, "peak_t_imad_eq": imad_peak / 1e12,
                                      "frac": e_ach / imad_peak},
            "binding_resource_ncu": ncu_pipes(rec),
            "imad_eq_speedup": all_ops * units / sec / imad_peak,
            "imad_eq_speedup_note": "all algorithmic word products as IMAD-eq / the INT32 IMAD peak: >1 means faster "
                                    "than any IMAD-only implementation could be (SURVEY §8(d) 'percent of IMAD peak')",
            "imad_eq_per_unit": all_ops}


def tcw_enabled():
    """the library's routing for k = 97 / 129 (mr_host.cpp tcw_enabled): tensor-core wide kernel unless switched off"""
    return os.environ.get("MR_RNS_IMAD_ONLY", "0") != "1" and os.environ.get("MR_RNS_TCW", "1") != "0"


def base_extension(wl):
    """which kernel family runs the workload's base extensions (the library routes by k: k <= 65 tensor
    path unless MR_RNS_IMAD_ONLY=1; k = 97 / 129 the tensor-core wide kernel unless MR_RNS_TCW=0)"""
    k = getattr(wl, "k", None) or 33
    if k >= 97:
        return ("tcgen05-i8 (k_modexp_tcw: base extensions and conversions on the tensor cores, images streamed by "
                "bulk copy)") if tcw_enabled() else "imad (k_modexp_wide, channels on threads)"
    return "imad" if os.environ.get("MR_RNS_IMAD_ONLY", "0") == "1" else "tcgen05-i8"


def kernel_name(wl):
    if isinstance(wl, MillerRabin):
        return "k_mr_rounds_tc (Miller-Rabin rounds, k=33, tcgen05 base extensions)"
    if isinstance(wl, Encrypt):
        if tcw_enabled():
            return "k_modexp_tcw (k=97, two 128-message tiles per SM, tcgen05 i8 contractions, TMA-streamed images)"
        return "k_modexp_wide (k=97 channels-on-threads, IMAD base extensions)"
    if os.environ.get("MR_RNS_IMAD_ONLY", "0") == "1":
        return "k_modexp (CRT half-ladders, IMAD-pipe base extensions)"
    return f"k_modexp_tc (CRT half-ladders, k={wl.k}, base extensions on tcgen05 int8)"


def workload_config(args, wl, total, world):
    cfg = {"workload": wl.describe, "units_total": total, "units_per_gpu": -(-total // world),
           "unit": wl.unit.replace("/s", ""),
           "base_extension": base_extension(wl),
           "inputs": "SplitMix64 by global index + edge values (synth/); identical for any GPU count",
           "l2": "flushed between timed steps (256 MiB write)"}
    if isinstance(wl, CrtDecrypt) or isinstance(wl, Encrypt):
        cfg["key"] = f"tests/golden/keys/{'rsa2048' if wl.L == 64 else 'rsa3072'}.json (oracle-generated)"
        cfg["modulus_bits"] = wl.key["n"].bit_length()
    if isinstance(wl, CrtDecrypt):
        cfg["rns_k_per_half"] = wl.k
    if args.total:
        cfg["strong_scaling_total"] = args.total
    return cfg


def ncu_record(name: str, count: int):
    """the committed ncu --set full summary of the ladder kernel in this configuration
    (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tensor = os.environ.get("MR_RNS_IMAD_ONLY", "0") != "1"
            return json.load(f).get(f"{'k_modexp_tc' if tensor else 'k_modexp'}/{name or 'c2'}/{count}")
    except (OSError, ValueError):
        return None


def ncu_pipes(rec):
    """utilisation of the CUDA-core resources from the same capture (issue slots, FMA-heavy pipe)."""
    if rec is None or "issue_active_pct" not in rec:
        return None
    return {k: rec[k] for k in ("issue_active_pct", "fmaheavy_pipe_pct", "alu_pipe_pct", "tensor_imma_pct",
                                "warp_instructions_per_multiplication", "source") if k in rec}


def cpu_baseline(wl: Workload, budget_s: float = 10.0):
    """the oracle, as it stands, on the host cores: a bounded sample of the same workload."""
    threads = os.cpu_count() or 1
    n = 64 * threads
    ins = wl.inputs(0, n)
    t0 = time.perf_counter()
    done = 0
    while True:
        wl.oracle(ins, threads)
        done += n
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": units_of(wl, done) / dt, "unit": wl.unit, "cores": threads, "cpu_model": cpu_model(),
            "kind": "oracle",
            "sample": f"{done} units of the same seeded workload (the first {n}, repeated) in {dt:.1f} s "
                      f"(oracle/oracle.c, {threads} pthreads)"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c2", "c3dec", "c3enc", "c5"], default="c2")
    ap.add_argument("--count", type=int, default=65536, help="units per GPU (weak scaling)")
    ap.add_argument("--total", type=int, default=0, help="total units over all GPUs (strong scaling)")
    ap.add_argument("--ref-sample", type=int, default=512, help="reference arm: units per step")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-identity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-multi", action="store_true", help="also time the oracle on rank 0 when N > 1")
    ap.add_argument("--dry-run-cpu", action="store_true")
    args = ap.parse_args(argv)
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        wl = make_workload(args.workload)
        wl.name = args.workload
        if args.dry_run_cpu:
            dev = CpuDryRun(wl)
            step = dev.step_fn()
        else:
            dev = CudaDevice(local)
            import paper_1305_3699_b200 as mr
            step = wl.make_device_step(mr, local)
        line = run_rank(args, world, rank, dev, wl, step)
        if line is not None:
            print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
