"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path of bench.py: contiguous
global-index sharding of the synthetic workload, the max-over-ranks timing reduction, and that the
union of the shards is byte-identical to the single-rank batch (messages are
independent, so sharding needs no data-path collective)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, count, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import oracle
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    key = bench.load_key("rsa1024")
    shard = synth.messages(key["n"], count, 0x5EEDC001, 32, edge=synth.edge_values(key["n"]), first=rank * count)
    # per-rank "step": the oracle stands in for the device work on this CPU-only box
    y = oracle.modexp_batch(shard, key["e"], key["n"])
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), y)
    t = bench.max_over_ranks(float(rank + 1) * 1.5, world)
    bench.barrier(world)
    with open(os.path.join(out_dir, f"max{rank}.txt"), "w") as f:
        f.write(repr(t))
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_rank(tmp_path):
    world, count = 2, 24
    port = _free_port()
    mp.spawn(_worker, args=(world, port, count, str(tmp_path)), nprocs=world, join=True)
    import bench
    import oracle
    import synth
    key = bench.load_key("rsa1024")
    full = synth.messages(key["n"], world * count, 0x5EEDC001, 32, edge=synth.edge_values(key["n"]))
    ref = oracle.modexp_batch(full, key["e"], key["n"])
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    assert np.array_equal(got, ref)
    for r in range(world):
        assert float(open(tmp_path / f"max{r}.txt").read()) == 3.0


def test_shard_inputs_independent_of_world_size():
    import bench
    import synth
    key = bench.load_key("rsa2048")
    a = synth.messages(key["n"], 64, 7, 64)
    b = np.concatenate([synth.messages(key["n"], 16, 7, 64, first=16 * r) for r in range(4)])
    assert np.array_equal(a, b)


def test_bench_numerator_matches_program_length():
    """the algorithmic numerator's mm count equals the best-window sliding-window count at the
    actual exponent (checked against an explicit window simulation at every w)."""
    import bench
    key = bench.load_key("rsa2048")
    for E in (key["dp"], key["dq"], 65537, 3, 1):
        best = None
        bits = E.bit_length()
        for w in range(1, 8):
            s = bin(E)[2:]
            # count windows left to right: zeros cost a squaring, a window of length L costs L squarings + 1 multiply
            i, n, first = 0, 0, True
            while i < len(s):
                if s[i] == "0":
                    n += 1
                    i += 1
                    continue
                j = min(i + w, len(s))
                while s[j - 1] == "0":
                    j -= 1
                if first:
                    first = False
                else:
                    n += (j - i) + 1
                i = j
            c = (2 ** (w - 1) if w > 1 else 0) + n
            best = c if best is None else min(best, c)
        assert bench.sliding_window_mm(E) == best + 2, E
        assert bits - 1 <= best <= 2 * bits
    per = bench.imad_eq_per_decrypt(key)
    assert 11.0e6 < per < 12.5e6            # 11.73 M IMAD-eq per RSA-2048 CRT decryption
