"""Per-kernel register / spill report of the last build (paper_1305_3699_b200/csrc/obj/*.log, ptxas -v)."""
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for log in sorted(glob.glob(os.path.join(ROOT, "paper_1305_3699_b200", "csrc", "obj", "*.o.log"))):
    name = None
    for line in open(log):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            raw = m.group(1)
            k = re.search(r"(k_[a-z0-9_]+?)(E|I|ILi)", raw)
            name = k.group(1) if k else raw[:60]
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            spill = (int(m.group(1)), int(m.group(2)))
        m2 = re.search(r"Used (\d+) registers", line)
        if m2 and name:
            if len(sys.argv) < 2 or spill != (0, 0):
                print(f"{os.path.basename(log):22s} {name:28s} regs {m2.group(1):>3s} spill st/ld {spill[0]}/{spill[1]}")
            name = None
