"""Parity-margin table from the GPU test session's record (tests/conftest.py `margin` fixture):
  python scripts/margins_table.py gpurun_out/parity_margins.json > profiles/r02/parity_margins.md
Every GPU parity assertion's measured error, its bound, and the ratio (1.0 = at the bound)."""
import json
import sys

rows = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_margins.json"))
rows.sort(key=lambda r: -(r["ratio"] or 0.0))
print("# GPU parity margins (measured error / bound; from `pytest -m gpu`, tests/conftest.py)\n")
print(f"{len(rows)} assertions; largest ratio first.\n")
print("| test | quantity | measured | bound | ratio |")
print("|---|---|---|---|---|")
for r in rows:
    t = r["test"].replace("tests/", "").replace("|", "/")
    print(f"| `{t}` | {r['what']} | {r['value']:.3g} | {r['bound']:.3g} | {r['ratio']:.3f} |")
