"""Summarise ncu reports / launch lists into markdown (run here, no GPU)."""
import csv, subprocess, sys, io, collections
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "smsp__average_warp_latency_issue_stalled_long_scoreboard", ]
def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    lines = []
    for row in r[2:]:
        d = dict(zip(h, row))
        lines.append(f"kernel `{d.get('Kernel Name','?')[:60]}`")
        for k in KEYS:
            if k in d:
                lines.append(f"- {k}: {d[k]} {units[h.index(k)]}")
    return "\n".join(lines)
def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for r in rows[start + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum": continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("tcg::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1e-3)
        tot[name] += v; cnt[name] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {100*v/T:.1f}% |")
    return "\n".join(lines)
if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"### {p}\n")
        print(report(p) if p.endswith(".ncu-rep") else launches(p))
        print()
