#!/bin/bash
# Build librte_b200.so in-tree (loads build.py directly, so a stale library never blocks the build).
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2604_23265_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); print(m.build())"
