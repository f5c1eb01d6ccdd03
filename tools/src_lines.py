"""Per-CUDA-source-line totals of an ncu report (instructions executed, stall
samples, shared wavefronts), from the `cuda,sass` source page.

    python tools/src_lines.py report.ncu-rep [top_n]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name") and r[0].isdigit():
        lines.append(r)
ix = {h: i for i, h in enumerate(hdr)}
S, E, W = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"], ix["L1 Wavefronts Shared"]
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
ts = sum(f(r[S]) for r in lines)
te = sum(f(r[E]) for r in lines)
tw = sum(f(r[W]) for r in lines)
print(f"samples {ts:.0f}  warp-instr {te/1e6:.1f}M  shared wavefronts {tw/1e6:.1f}M")
agg = {}
for r in lines:
    key = int(r[0])
    a = agg.setdefault(key, [0.0, 0.0, 0.0, r[1]])
    a[0] += f(r[S]); a[1] += f(r[E]); a[2] += f(r[W])
for k, (s, e, w, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:5d} {100*s/ts:5.1f}%s {100*e/te:5.1f}%i {100*w/max(tw,1):5.1f}%w  {src.strip()[:90]}")


def ranges(spec):
    """spec: name=a-b,... -> instruction / sample / wavefront share per line range"""
    out = []
    for item in spec.split(","):
        name, r = item.split("=")
        a, b = (int(x) for x in r.split("-"))
        s = sum(v[0] for k, v in agg.items() if a <= k <= b)
        e = sum(v[1] for k, v in agg.items() if a <= k <= b)
        w = sum(v[2] for k, v in agg.items() if a <= k <= b)
        out.append((name, s / ts, e / te, w / max(tw, 1)))
    return out


if len(sys.argv) > 3:
    for name, s, e, w in ranges(sys.argv[3]):
        print(f"{name:>12}: samples {100*s:5.1f}%  instr {100*e:5.1f}%  wavefronts {100*w:5.1f}%")
