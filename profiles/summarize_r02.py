"""Round-2 profile summaries from a tools/ncu_kernels.sh capture directory.

    python profiles/summarize_r02.py gpurun_out/<tag> [more dirs ...]

Reads raw_{inv,visc,viscstage}_N<n>.csv (ncu --set full --page raw --csv, one
launch each on the 1000x1000 wavy mesh) and writes

  profiles/r02_ncu_traffic.json   per configuration: duration, DRAM bytes per
                                  launch against the algorithmic bytes of that
                                  launch, pipe use, occupancy, stall mix; keys
                                  inv_N<n> (stage kernel, a stage-2 launch) and
                                  visc_N<n> (viscous pre-kernel + viscous stage
                                  kernel of one stage), which bench.py reports
  profiles/r02_ncu_stage_sweep.txt  the same as a table

Algorithmic bytes per node: a stage-2 launch of the inviscid stage
kernel moves 120 B (state 24 + W^n 24 + 6 geometry fields 48 + state out 24); the
viscous pre-kernel reads state + 4 metrics + J (64 B) and writes the 4 flux
pairs (32 B); the viscous stage kernel is the inviscid one plus the 4 flux
pairs read (32 B)."""
import csv
import json
import os
import sys

DST = os.path.dirname(os.path.abspath(__file__))
KX = 1000
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
ALG = {"inv": 120.0, "visc": 96.0, "viscstage": 152.0}


def raw(path):
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


def summary(d, kind, N):
    nodes = KX * KX * (N + 1) ** 2
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and isinstance(v, float)}
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    return {
        "kernel": str(d.get("Kernel Name", ""))[:60],
        "time_us": d["gpu__time_duration.sum"],
        "dram_bytes_per_launch": dram,
        "algorithmic_bytes_per_launch": ALG[kind] * nodes,
        "traffic_over_algorithmic": dram / (ALG[kind] * nodes),
        "dram_pct": d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "fp64_pipe_pct": d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "warps_per_sm": d.get("sm__warps_active.avg.per_cycle_active"),
        "registers": d.get("launch__registers_per_thread"),
        "stalls": {k: round(100 * v / tot, 1) for k, v in top},
    }


def main():
    out = {}
    for src in sys.argv[1:]:
        for f in sorted(os.listdir(src)):
            if not (f.startswith("raw_") and f.endswith(".csv")):
                continue
            kind, n = f[4:-4].rsplit("_N", 1)
            try:
                out[f"{kind}_N{int(n)}"] = summary(raw(os.path.join(src, f)), kind, int(n))
            except Exception as e:  # an incomplete capture
                print("skip", f, e)
    # one viscous stage = pre-kernel + stage kernel
    for key in [k for k in out if k.startswith("visc_N")]:
        n = key[6:]
        s = out.get(f"viscstage_N{n}")
        if s:
            pre = out[key]
            out[key] = {"kernel": pre["kernel"] + " + " + s["kernel"],
                        "time_us": pre["time_us"] + s["time_us"],
                        "dram_bytes_per_launch": pre["dram_bytes_per_launch"] + s["dram_bytes_per_launch"],
                        "algorithmic_bytes_per_launch": pre["algorithmic_bytes_per_launch"]
                        + s["algorithmic_bytes_per_launch"],
                        "pre_kernel": pre, "stage_kernel": s}
            out[key]["traffic_over_algorithmic"] = (out[key]["dram_bytes_per_launch"]
                                                    / out[key]["algorithmic_bytes_per_launch"])
    with open(os.path.join(DST, "r02_ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    lines = ["# ncu --set full, one launch per configuration, 1000x1000 wavy mesh (1M elements), "
             "B200, cold L2",
             "config          time_us  dram_GB  alg_GB  traffic/alg  DRAM%  FP64%  warps  regs  "
             "top stalls"]
    for k in sorted(out, key=lambda k: (k.split("_N")[0], int(k.split("_N")[1]))):
        s = out[k]
        parts = [s] if "pre_kernel" not in s else [s["pre_kernel"], s["stage_kernel"]]
        for p in parts:
            lines.append(f"{k:14s} {p['time_us']:9.1f} {p['dram_bytes_per_launch'] / 1e9:8.3f} "
                         f"{p['algorithmic_bytes_per_launch'] / 1e9:7.3f} "
                         f"{p['traffic_over_algorithmic']:11.2f} {p['dram_pct'] or 0:6.1f} "
                         f"{p['fp64_pipe_pct'] or 0:6.1f} {p['warps_per_sm'] or 0:6.1f} "
                         f"{int(p['registers'] or 0):5d}  "
                         + ", ".join(f"{a} {b}%" for a, b in p["stalls"].items())
                         + f"   [{p['kernel']}]")
    with open(os.path.join(DST, "r02_ncu_stage_sweep.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
