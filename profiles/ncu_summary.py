"""Summarise an ncu report (raw page): the metrics the roofline and the stall
analysis cite.  Usage: python profiles/ncu_summary.py report.ncu-rep [out.txt]"""
import csv
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hdr, units = rows[0], rows[1]
    lines = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '')[:100]}")
        for k in KEEP:
            if k in d:
                lines.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
        st = []
        for h, v in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    st.append((float(v), h))
                except ValueError:
                    pass
        lines.append("# top stall reasons (pc samples)")
        for v, h in sorted(st, reverse=True)[:8]:
            lines.append(f"{h} = {int(v)}")
    return "\n".join(lines)


if __name__ == "__main__":
    text = summarize(sys.argv[1])
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(text + "\n")
    print(text)
