"""Summarise an ncu report (or a launch-list CSV) into a text file under profiles/.

    python scripts/summarize_ncu.py report.ncu-rep > profiles/<name>.txt
    python scripts/summarize_ncu.py launches.csv > profiles/<name>.txt
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst issue % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU wavefronts % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:110]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:32s} {d[k]:>16s} {u.get(k, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * scale[u["dram__bytes_read.sum"]] + wr * scale[u["dram__bytes_write.sum"]]
            print(f"  {'traffic (read+write) bytes':32s} {tot:16.4e}")
        except (KeyError, ValueError):
            pass
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        print("  warp stall samples: " + ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in sorted(stalls, reverse=True)[:6]))
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    mult = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * mult.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'total us':>12s} {'share':>6s} {'launches':>8s} {'avg us':>9s}  kernel  (ncu --metrics gpu__time_duration.sum: "
          "cold-cache, serialised; compare shares)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:12.1f} {100 * t / tot:5.1f}% {n:8d} {t / n:9.2f}  {k}")
    print(f"{tot:12.1f} total")


if __name__ == "__main__":
    p = sys.argv[1]
    (report if p.endswith(".ncu-rep") else launches)(p)
