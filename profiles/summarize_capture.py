"""Turn a profiles/capture.sh run (gpurun_out/prof_r01/) into the committed
profile summaries:

  profiles/r01_ncu_traffic.json   per degree: the stage kernel's duration, DRAM
                                  bytes per launch (ncu, cold L2) against the
                                  algorithmic bytes, pipe use, occupancy, stalls
  profiles/r01_ncu_stage_sweep.txt  the same as a table
  profiles/r01_launches_n7.txt    the ncu launch list of the bench command
  profiles/r01_bench_n7.json      the bench line
  profiles/r01_sweep.txt          N=1..15 stage times (CUDA events, warm)

The captured launch is the second stage kernel of the run (-s 1: SSPRK3 stage 2,
which reads W^n: 120 algorithmic bytes per node)."""
import csv
import json
import os
import re
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_r01"
DST = os.path.dirname(os.path.abspath(__file__))
KX = 1000


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def raw(path):
    """ncu --page raw --csv -> {metric: value in base units (bytes, microseconds)}"""
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[i], rows[i + 1], rows[i + 2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
        except ValueError:
            d[h] = v
    return d


def num(d, k):
    v = d.get(k)
    return v if isinstance(v, float) else None


def main():
    out, lines = {}, []
    lines.append("N  kernel                 time_us  dram_GB  alg_GB  traffic/alg  DRAM%  FP64pipe%  "
                 "warps/SM  regs  top stalls")
    for N in range(1, 16):
        p = os.path.join(SRC, f"ncu_n{N}_raw.csv")
        if not os.path.exists(p):
            continue
        try:
            d = raw(p)
        except Exception:
            continue
        n1 = N + 1
        nn = KX * KX * n1 * n1
        t_us = num(d, "gpu__time_duration.sum")
        rd_b, wr_b = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
        stalls = sorted(((num(d, k) or 0.0, k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled")
                         and not k.endswith("not_issued")), reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        top = [(k, round(100 * v / tot, 1)) for v, k in stalls[:5]]
        alg = 120.0 * nn
        e = {"kernel": d.get("Kernel Name", "")[:80],
             "duration_us": t_us,
             "dram_bytes_per_launch": (rd_b or 0) + (wr_b or 0),
             "dram_read_bytes": rd_b, "dram_write_bytes": wr_b,
             "algorithmic_bytes_per_launch": alg,
             "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "fp64_pipe_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "warps_active_per_sm": num(d, "sm__warps_active.avg.per_cycle_active"),
             "registers": num(d, "launch__registers_per_thread"),
             "inst_executed": num(d, "smsp__inst_executed.sum"),
             "top_stalls_pct": top}
        out[f"inv_N{N}"] = e
        name = re.sub(r"^void |\(.*", "", e["kernel"]).replace("swdg_dev::", "").replace(
            "<unnamed>::", "")
        lines.append(f"{N:<2} {name[:22]:<22} {t_us or 0:8.1f} {e['dram_bytes_per_launch'] / 1e9:8.3f} "
                     f"{alg / 1e9:7.3f} {e['dram_bytes_per_launch'] / alg:11.2f}  "
                     f"{e['dram_throughput_pct'] or 0:5.1f}  {e['fp64_pipe_pct'] or 0:9.1f}  "
                     f"{e['warps_active_per_sm'] or 0:8.1f}  {int(e['registers'] or 0):4d}  "
                     + ", ".join(f"{k} {v}%" for k, v in top[:3]))
    with open(os.path.join(DST, "r01_ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(DST, "r01_ncu_stage_sweep.txt"), "w") as f:
        f.write("# ncu --set full, one stage-kernel launch (SSPRK3 stage 2) per degree, 1000x1000 wavy "
                "mesh (1M elements), B200, cold L2 (ncu cache control)\n")
        f.write("\n".join(lines) + "\n")
    # launch list
    p = os.path.join(SRC, "launches_n7.csv")
    if os.path.exists(p):
        rows = [r for r in csv.reader(open(p)) if r and r[0] != "ID" and len(r) > 14]
        per = {}
        for r in rows:
            if r[12] != "gpu__time_duration.sum":
                continue
            name = re.sub(r"\(.*", "", r[4])
            v = float(r[14].replace(",", ""))
            per.setdefault(name, []).append(v)
        tot = sum(sum(v) for v in per.values()) or 1.0
        with open(os.path.join(DST, "r01_launches_n7.txt"), "w") as f:
            f.write("# ncu launch list of `python bench.py --steps 2 --warmup 3 --cpu-budget 1 --no-sweep` (N=7, "
                    "1M elements): gpu__time_duration per kernel, serialised, cold\n")
            f.write("kernel\tlaunches\tavg\tsum\tshare\n")
            for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{name}\t{len(v)}\t{sum(v) / len(v):.1f}\t{sum(v):.1f}\t{sum(v) / tot:.3f}\n")
    for a, b in (("bench_n7.json", "r01_bench_n7.json"), ("sweep.txt", "r01_sweep.txt"),
                 ("sweep_visc.txt", "r01_sweep_visc.txt"),
                 ("bench_n7_visc.json", "r01_bench_n7_visc.json"),
                 ("bench_n7_dist1.json", "r01_bench_n7_dist1.json"),
                 ("bench_ref.json", "r01_bench_ref.json")):
        p = os.path.join(SRC, a)
        if os.path.exists(p):
            with open(p) as fi:
                lines = fi.read().splitlines()
            if a.endswith(".json"):  # the bench line (drop any banner before it)
                lines = [l for l in lines if l.startswith("{")][-1:]
            with open(os.path.join(DST, b), "w") as fo:
                fo.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
