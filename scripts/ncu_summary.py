"""Summarise ncu outputs: per-kernel launch shares from a --csv launch list
and key metrics from a --set full report."""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:34s} n={n:6d} total={t:10.1f}us avg={t / n:8.2f}us share={t / tot:.3f}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct", "smsp__warp_issue_stalled_membar_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct", "smsp__warp_issue_stalled_wait_per_warp_active.pct"]


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        vals = []
        for k in KEYS:
            if k in h:
                vals.append(f"{k.split('.')[0].replace('smsp__warp_issue_stalled_', 'stall_')}={r[h.index(k)]}{units[h.index(k)]}")
        out.append(name + ": " + ", ".join(vals))
    return "\n".join(out)


def traffic(path, kernels=("k_rowdot", "k_zreduce", "k_coltile")):
    """DRAM bytes (read + write) of one 3-axis solve: the first capture of each
    solve kernel in a --set full report, summed."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    seen = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        base = name.split("<")[0]
        if base in kernels and base not in seen:
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(r[h.index(k)].replace(",", "")) * scale[units[h.index(k)]]
            seen[base] = b
    return seen


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        import json
        per = traffic(sys.argv[2])
        print(json.dumps({"traffic_bytes_per_solve": sum(per.values()), "per_kernel_bytes": per,
                          "source": sys.argv[2]}, indent=1))
        sys.exit(0)
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(launches(p) if p.endswith(".csv") else report(p))
