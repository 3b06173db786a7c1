"""Aggregate ncu per-SASS-line stall samples and executed instructions over line ranges
(experiments): python scripts/ncu_regions.py report.ncu-rep a-b [c-d ...]; with no ranges, prints
runs of lines sharing one execution count (a proxy for code regions / roles)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia = h.index("Instructions Executed")
isrc = h.index("Source")
stalls = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def region(a, b):
    tot = {h[i]: 0.0 for i in stalls}
    inst = 0.0
    for r in data[a:b + 1]:
        inst += f(r[ia])
        for i in stalls:
            tot[h[i]] += f(r[i])
    s = sum(tot.values())
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
    print(f"lines {a}-{b}: inst {inst:.0f} samples {s:.0f} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in top))


if len(sys.argv) > 2:
    for rg in sys.argv[2:]:
        a, b = map(int, rg.split("-"))
        region(a, b)
else:
    runs = []
    cur = None
    for k, r in enumerate(data):
        c = f(r[ia])
        if cur and c == cur[2]:
            cur[1] = k
        else:
            if cur:
                runs.append(cur)
            cur = [k, k, c]
    runs.append(cur)
    for a, b, c in runs:
        if b - a >= 8 and c > 0:
            region(a, b)
