"""Per-source-line dynamic instruction and stall-sample shares of one kernel from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTRING [top]

Joins ncu's SASS page (instructions executed, warp-stall samples per SASS address) with the line
table of the same object (nvdisasm -g), so the counts map to mr_kernels.cuh lines."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, kern, top=40):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
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
        m = re.search(r'//## File "(.*?)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    base = int(data[0]["Address"], 16)
    inst, samp = collections.Counter(), collections.Counter()
    opc = os.environ.get("OPCODE")   # e.g. OPCODE=IMAD.WIDE.U32: count only that SASS opcode
    for d in data:
        if opc and d["Source"].split()[0 if not d["Source"].startswith("@") else 1] != opc:
            continue
        ln = off2line.get(int(d["Address"], 16) - base)
        inst[ln] += int(d["Instructions Executed"] or 0)
        samp[ln] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    ti, ts = sum(inst.values()), max(1, sum(samp.values()))
    csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1305_3699_b200", "csrc")
    srcs = {}

    def text(key):
        if not key:
            return ""
        f, ln = key
        if f not in srcs:
            path = os.path.join(csrc, f)
            srcs[f] = open(path).read().splitlines() if os.path.exists(path) else []
        return srcs[f][ln - 1].strip()[:90] if ln <= len(srcs[f]) else ""
    print(f"total warp-instructions {ti:,}  stall samples {ts:,}")
    for key, c in inst.most_common(int(top)):
        where = f"{key[0]}:{key[1]}" if key else "?"
        print(f"{where:>22} {100 * c / ti:5.1f}% inst {100 * samp[key] / ts:5.1f}% samp | {text(key)}")


if __name__ == "__main__":
    main(*sys.argv[1:])
