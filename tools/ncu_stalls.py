"""Per-source-line warp-stall samples of one kernel by stall reason, from ncu's SASS source page.

    python tools/ncu_stalls.py SASS.csv OBJ.o KERNEL_SUBSTRING REASON [top]

SASS.csv = `ncu -i REPORT --page source --csv --print-source sass`; REASON e.g. stall_long_sb."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, kern):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    lines = sass.splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l][0]
    cur, off2line = None, {}
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File ".*?", line (\d+)', l)
        if m:
            cur = int(m.group(1))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    return off2line


def main(csvf, obj, kern, reason, top=25):
    rows = list(csv.reader(open(csvf)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
    o2l = line_map(obj, kern)
    base = int(data[0]["Address"], 16)
    c = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    for d in data:
        ln = o2l.get(int(d["Address"], 16) - base)
        v = int(d.get(reason) or 0)
        c[ln] += v
        ops[ln][re.sub(r'^@!?U?P\w+\s+', '', d["Source"].strip()).split(' ')[0]] += v
    tot = sum(c.values())
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_1305_3699_b200", "csrc", "mr_kernels.cuh")).read().splitlines()
    print(f"{reason}: {tot:,} samples")
    for ln, v in c.most_common(int(top)):
        o = ",".join(f"{k}:{n}" for k, n in ops[ln].most_common(2))
        print(f"{ln!s:>5} {100 * v / max(tot, 1):5.1f}% [{o}] | {src[ln - 1].strip()[:80] if ln else ''}")


if __name__ == "__main__":
    main(*sys.argv[1:])
