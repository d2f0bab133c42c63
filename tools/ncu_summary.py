"""Summarise an ncu report (.ncu-rep) into the text kept under profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--algo-bytes B] > profiles/rNN_x.txt

Per kernel: duration, DRAM/L2 traffic and throughput, LSU (L1TEX data pipe)
utilisation split into shared/global, bank conflicts, occupancy limits, the
top warp-stall reasons, and -- when --algo-bytes is given -- achieved
algorithmic GB/s for the kernel.
"""
import argparse
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % peak"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "LSU wavefronts % peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "  of which shared % peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs), blocks"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem), blocks"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--algo-bytes", type=float, default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    for d in data:
        print(f"== {d[ix['Kernel Name']][:110]}")
        for k, label in KEYS:
            if k in ix and d[ix[k]] != "":
                print(f"  {label:34s} {d[ix[k]]} {units[ix[k]]}")
        if a.algo_bytes and "gpu__time_duration.sum" in ix:
            t = float(d[ix["gpu__time_duration.sum"]])
            unit = units[ix["gpu__time_duration.sum"]]
            sec = t * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1e-6)
            print(f"  {'algorithmic GB/s (cold, this launch)':34s} {a.algo_bytes / sec / 1e9:.1f}")
        pre = "smsp__pcsamp_warps_issue_stalled_"
        st = [(h[len(pre):], float(d[i] or 0)) for i, h in enumerate(hdr)
              if h.startswith(pre) and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        top = sorted(st, key=lambda t: -t[1])[:6]
        print("  top stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in top))
    return 0


if __name__ == "__main__":
    sys.exit(main())
