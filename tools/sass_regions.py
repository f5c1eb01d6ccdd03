"""Summarise an ncu SASS source page (csv) into regions between barriers."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
i_w = hdr.index("L1 Wavefronts Shared")
i_wi = hdr.index("L1 Wavefronts Shared Ideal")
tot_s = sum(float(r[i_s] or 0) for r in data)
tot_e = sum(float(r[i_e] or 0) for r in data)
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_e/1e6:.1f}M")
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
start = 0
acc_s = acc_e = 0.0
for k, r in enumerate(data):
    s = float(r[i_s] or 0)
    e = float(r[i_e] or 0)
    acc_s += s
    acc_e += e
    src = r[i_src]
    mark = any(t in src for t in ("BAR.SYNC", "EXIT", "ATOMS", "STG", "STS", "RET"))
    if s / tot_s > thr or "BAR.SYNC" in src or "ATOMS" in src or "STG" in src:
        w = f"{r[i_w]}/{r[i_wi]}" if r[i_w] not in ("", "0") else ""
        print(f"{k:5d} {100*s/tot_s:5.1f}% {100*e/tot_e:5.1f}%i {w:>22}  {src[:80]}")
    if "BAR.SYNC" in src:
        print(f"      ---- region {start}-{k}: samples {100*acc_s/tot_s:.1f}%  instr {100*acc_e/tot_e:.1f}%")
        start = k + 1
        acc_s = acc_e = 0.0
print(f"      ---- region {start}-end: samples {100*acc_s/tot_s:.1f}%  instr {100*acc_e/tot_e:.1f}%")
