"""List SASS instructions of an ncu report in [a, b) with execution counts."""
import csv, subprocess, sys
rep, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
minc = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
i_src = hdr.index("Source"); i_e = hdr.index("Instructions Executed")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
tot = 0
for k in range(a, min(b, len(data))):
    r = data[k]; e = float(r[i_e] or 0); tot += e
    if e / 1e6 >= minc:
        print(k, f"{e/1e6:8.2f}M", r[i_s], r[i_src][:90])
print(f"sum {tot/1e6:.1f}M")
