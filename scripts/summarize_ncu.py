#!/usr/bin/env python
"""Summarise ncu outputs into small text files for profiles/.

  python scripts/summarize_ncu.py launches <launches.csv> > profiles/rNN/launches_summary.txt
  python scripts/summarize_ncu.py full <prof.ncu-rep> > profiles/rNN/<kernel>_full.txt

`launches`: per-kernel device time from the `--metrics gpu__time_duration.sum` pass (cold-cache,
serialised: compare SHARES, not absolutes).  `full`: the key roofline metrics of each captured
launch of a `--set full` report (DRAM bytes, throughput, tensor/FMA pipe, occupancy).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("rte::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return name.strip()


def launches(path):
    with open(path) as f:
        lines = f.read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        ns = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            ns *= 1e3
        elif r["Metric Unit"] == "ms":
            ns *= 1e6
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"# ncu launch list: {len(rows)} launches, total {tot / 1e6:.3f} ms (cold-cache, serialised)")
    print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'avg_us':>9s}")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {n:8d} {ns / 1e6:10.3f} {ns / tot:7.3f} {ns / n / 1e3:9.1f}")


FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        print(f"## {short(r[hdr.index('Kernel Name')])}")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:66s} {r[i]:>16s} {units[i]}")


def table(path):
    """One line per captured launch of a `full` summary file (this script's own output): duration, tensor
    pipe activity, DRAM bytes, grid -- e.g. every GEMM of one V-cycle in launch order."""
    rows, cur = [], None
    for line in open(path):
        if line.startswith("## "):
            cur = {"k": line[3:].strip().replace("void gemm3xtf32_kernel", "gemm3xtf32")}
            rows.append(cur)
        elif cur is not None and line.startswith("  "):
            parts = line.split()
            cur[parts[0]] = (float(parts[1].replace(",", "")), parts[2] if len(parts) > 2 else "")
    print(f"# {len(rows)} launches of {path} (ncu --set full: serialised, cold-cache; template arguments = "
          "<N tile, A mode (1 = halo), pre-split A, epilogue, CTAs per SM>)")
    print(f"{'#':>3s} {'kernel':40s} {'grid':>5s} {'us':>8s} {'tensor%':>8s} {'dram_rd_MB':>11s} {'dram_wr_MB':>11s}")
    for i, r in enumerate(rows):
        t, u = r.get("gpu__time_duration.sum", (0.0, "us"))
        t *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
        mb = lambda k: r.get(k, (0.0, ""))[0] * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(r.get(k, (0, "Mbyte"))[1], 1.0)
        print(f"{i:3d} {r['k'][:40]:40s} {int(r.get('launch__grid_size', (0, ''))[0]):5d} {t:8.1f} "
              f"{r.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', (0, ''))[0]:8.1f} "
              f"{mb('dram__bytes_read.sum'):11.1f} {mb('dram__bytes_write.sum'):11.1f}")


if __name__ == "__main__":
    {"launches": launches, "full": full, "table": table}[sys.argv[1]](sys.argv[2])
