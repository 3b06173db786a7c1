"""Per-launch DRAM traffic of the Arnoldi kernels over the timed bench steps -> profiles/traffic.json
(bench.py reports it as roofline.traffic for the dominant class).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"cgs_kernel|dcgs_update_kernel" --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      > gpurun_out/cgs_traffic.csv
  python scripts/traffic.py gpurun_out/cgs_traffic.csv 30 > profiles/traffic.json

Template arguments of cgs_kernel<T, NV, UPDATE, DOTS> name the timing class (csrc/krylov.cu):
UPDATE && DOTS = cgs_update_dots, DOTS only = cgs_dots, UPDATE only = cgs_update;
dcgs_update_kernel<T, NV> is dcgs_update.  The last `steps` launches of each class (one per GMRES
step: a whole restart cycle = 30) are averaged, so the figure is per launch over every j of a cycle,
the same average the bench's roofline takes."""
import collections
import csv
import io
import json
import re
import sys

path, steps = sys.argv[1], int(sys.argv[2])
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
per = collections.OrderedDict()
for r in rows:
    per.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
unit = {}
for r in rows:
    unit[r["Metric Name"]] = r["Metric Unit"]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
classes = collections.defaultdict(list)
for v in per.values():
    if "dcgs_update_kernel" in v["name"]:
        cls = "dcgs_update"
    else:
        m = re.search(r"cgs_kernel<[^,]+,\s*\d+,\s*(\d+),\s*(\d+)>", v["name"])
        if not m:
            continue
        upd, dots = int(m.group(1)), int(m.group(2))
        cls = "cgs_update_dots" if upd and dots else ("cgs_dots" if dots else "cgs_update")
    b = v.get("dram__bytes_read.sum", 0) * scale[unit["dram__bytes_read.sum"]] + \
        v.get("dram__bytes_write.sum", 0) * scale[unit["dram__bytes_write.sum"]]
    classes[cls].append(b)
out = {c: sum(b[-steps:]) / len(b[-steps:]) for c, b in classes.items() if b}
out["_source"] = "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over the last %d launches of each class" % steps
print(json.dumps(out, indent=1))
