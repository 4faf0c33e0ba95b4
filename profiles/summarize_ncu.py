"""Extract the judged metrics from an `ncu --set full` report into a text summary.

usage: python profiles/summarize_ncu.py report.ncu-rep [kernel-regex]
(reads `ncu -i <rep> --page raw --csv`; needs the ncu CLI, no GPU)
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")


def main(rep, kregex=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        rec = dict(zip(hdr, vals))
        name = rec.get("Kernel Name", "")
        if kregex and not re.search(kregex, name):
            continue
        print(f"== {name[:160]}")
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k:
                    print(f"  {k:70s} {vals[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            m = STALL.fullmatch(h)
            if m:
                try:
                    stalls.append((float(vals[i]), m.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stall reasons (warps per issue):",
              ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
        for i, h in enumerate(hdr):
            if re.search(r"pipe_(tc|tensor|tmem|uniform|xu|fma|alu)\w*\.avg\.pct_of_peak_sustained_active$", h) \
                    and h not in KEYS:
                print(f"  {h:70s} {vals[i]:>16s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
