"""Summarise ncu outputs into profiles/ (run here, after gpurun brought them back).

  python tools/summarize_ncu.py launches gpurun_out/launches_r1.csv > profiles/r1_launches.md
  python tools/summarize_ncu.py full gpurun_out/prof512_r1.ncu-rep > profiles/r1_kernels_512.md
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        ms = float(r[ix["Metric Value"]].replace(",", "")) * UNIT[r[ix["Metric Unit"]]]
        a = agg.setdefault(name, [0, 0.0, r[ix["Grid Size"]], r[ix["Block Size"]]])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {path}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised;"
          " compare shares, not absolutes)\n")
    print("| kernel | launches | total ms | ms/launch | share | grid | block |")
    print("|---|---|---|---|---|---|---|")
    for k, (n, t, gs, bs) in agg.items():
        print(f"| `{k}` | {n} | {t:.2f} | {t / n:.3f} | {100 * t / tot:.1f}% | {gs} | {bs} |")


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs), CTAs"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem), CTAs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long sb / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short sb / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full: {path}\n")
    names = []
    for r in rows[2:]:
        names.append(r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("mxb::", ""))
    print("| metric | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in ix:
            continue
        vals = [r[ix[key]] for r in rows[2:]]
        print(f"| {label} ({units[ix[key]]}) | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
