"""Summarises ncu reports / launch lists into profiles/ (committed evidence).

    python scripts/ncu_summary.py gpurun_out/X.ncu-rep [...]  -> prints key metrics
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv -> per-kernel share table
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_registers",
        "sm__maximum_warps_per_active_cycle_pct"]


SETUP = {"factor_level_kernel", "assemble_kernel", "forward_panel_kernel", "backward_panel_kernel", "volume_kernel",
         "face_kernel", "k0_kernel"}


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel: {name[:120]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k} = {r[i]} {units[i]}")
    return "\n".join(lines)


def launches(path):
    text = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(text))
    hdr = rows[0]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
        tot[name] += float(r[hdr.index("Metric Value")]) / 1e3
        cnt[name] += 1
    # one-time setup kernels (device factorisation / panel formation) are
    # listed apart; shares are of the time-step kernels only
    setup = {k for k in tot if k in SETUP}
    total = sum(v for k, v in tot.items() if k not in setup)
    lines = [f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share of steps':>14s}"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if k in setup:
            continue
        lines.append(f"{k:28s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:8.2f} {v / total:14.1%}")
    if setup:
        lines.append("setup (once per simulation, not in the steps):")
        for k in sorted(setup, key=lambda k: -tot[k]):
            lines.append(f"  {k:26s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k] / cnt[k]:8.2f}")
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for p in sys.argv[1:]:
            print(rep(p))
