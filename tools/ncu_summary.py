"""Key metrics of ncu --set full reports: python tools/ncu_summary.py REPORT.ncu-rep ..."""
import csv, subprocess, sys
def summ(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (x + (" " + y if y and y != "%" else "")) for k, y, x in zip(h, u, v)}
    keys = {"kernel": "Kernel Name", "ms": "gpu__time_duration.sum", "dram_rd_GB": "dram__bytes_read.sum",
            "dram_wr_GB": "dram__bytes_write.sum", "issue%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
            "fmaheavy%": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fma%": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "alu%": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "tensor%": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
            "smem_per_block": "launch__shared_mem_per_block_dynamic"}
    r = {}
    for k, m in keys.items():
        cands = [x for x in h if x == m] or [x for x in h if x.endswith(m)]
        r[k] = d.get(cands[0], "?") if cands else "?"
    raw = dict(zip(h, v))
    stalls = {x.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(raw[x] or 0) for x in h
              if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1
    top = sorted(stalls.items(), key=lambda t: -t[1])[:7]
    r["top_stalls"] = ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in top)
    return r
for rep in sys.argv[1:]:
    print(rep, summ(rep))
