"""Summarise a MR_TCW_TRACE timeline (mr_tcw.cuh WTrace): per (tile, role) region, the mean cycles between
consecutive events, grouped by transition.      python tools/tcw_trace.py FILE [tile]"""
import collections
import sys

import numpy as np

W_TRN = 2700
raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16384)[-1]
want_tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
names = {0: "BE1", 1: "BE2", 2: "TRN", 3: "EXT"}


def name(c):
    role, e = (c >> 8) & 0xF, c & 0xFF
    if role == 1:
        return f"MMA {names[(e >> 4) & 0xF]} " + ["aready", "acce", "issued", "full"][e & 0xF]
    if role == 2:
        return f"PRD {names[(e >> 4) & 0xF]} " + ["?", "slab0", "slab"][e & 0xF]
    if e == 0x0E:
        return "cmp mult-start"
    if e == 0x0F:
        return "cmp a_done"
    return f"cmp {names[(e >> 4) & 0xF]} " + {1: "accf", 2: "released", 3: "epi-done"}[e & 0xF]


for role in range(3):
    base = 1 + (want_tile * 3 + role) * W_TRN
    recs = raw[base:base + W_TRN]
    recs = recs[recs != 0]
    if not len(recs):
        continue
    clk = (recs >> np.uint64(16)).astype(np.int64)
    code = (recs & np.uint64(0xFFFF)).astype(np.int64)
    print(f"== tile {want_tile} role {role}: {len(recs)} events over {clk[-1] - clk[0]:,} cycles")
    gaps = collections.defaultdict(list)
    for i in range(1, len(clk)):
        gaps[(name(code[i - 1]), name(code[i]))].append(clk[i] - clk[i - 1])
    for (a, b), v in sorted(gaps.items(), key=lambda x: -sum(x[1]))[:16]:
        print(f"{sum(v)/1e3:10.1f}k  n={len(v):5d} mean={np.mean(v):8.0f}  {a}  ->  {b}")
