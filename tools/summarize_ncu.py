"""Summarise ncu outputs into text for profiles/ (run here, no GPU needed).

    python tools/summarize_ncu.py launches <csv>         # per-kernel share of a launch list
    python tools/summarize_ncu.py full <ncu-rep>          # key metrics per captured launch
"""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    t = defaultdict(float)
    n = defaultdict(int)
    for r in rows:
        k = r[4]
        t[k] += float(r[-1]) / 1e6
        n[k] += 1
    tot = sum(t.values())
    print(f"launch list {path}: {len(rows)} launches, {tot:.3f} ms total device time "
          "(ncu, serialised, cold caches: compare shares, not absolutes)")
    for k in sorted(t, key=t.get, reverse=True):
        print(f"  {100*t[k]/tot:6.2f}%  n={n[k]:5d}  avg {t[k]/n[k]:8.4f} ms  {k[:90]}")


KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"ncu --set full capture {path}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"\n== {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {r[i]:>20s} {units[i]}")
        if "dram__bytes_read.sum" in hdr:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(k)
                tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
            print(f"  traffic (dram read+write) = {tot:.4e} bytes per launch")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
