#!/bin/bash
# Round-2 measurement set on one B200 (run through gpurun from the repo root); every file lands in
# gpurun_out/r02/ and the kept ones are copied to profiles/r02/ (profiles/README.md says which is which).
# Timed runs first, ncu afterwards (a number printed under ncu is never a bench value).
set -u
O=gpurun_out/r02
mkdir -p $O
run() { echo "== $*" >&2; "$@"; echo "rc $?" >&2; }
if [ "${PART:-all}" = "bench" ] || [ "${PART:-all}" = "all" ]; then
  run python bench.py --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
  for k in 1 2 3; do run python bench.py --config $k --steps 5 --warmup 3 > $O/bench_cfg$k.json 2> $O/bench_cfg$k.err; done
  run python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
  run python bench.py --steps 5 --warmup 3 --coeffnet --no-cpu-baseline > $O/bench_cfg5_coeffnet.json 2> $O/bench_cfg5_coeffnet.err
  run python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
  for k in 1 2 3 5; do run python bench.py --time-to-tol --config $k > $O/time_to_tol_cfg$k.json 2> $O/time_to_tol_cfg$k.err; done
  run python scripts/tfps_bench.py > $O/tfps_cfg2.json 2> $O/tfps_cfg2.err
  run python scripts/paper_workload.py > $O/paper_workload.json 2> $O/paper_workload.err
fi
if [ "${PART:-all}" = "ncu" ] || [ "${PART:-all}" = "all" ]; then
  NCU=/usr/local/cuda/bin/ncu
  run $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
  run $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"cgs_kernel|dcgs_update_kernel" --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      > $O/cgs_traffic.csv 2> $O/cgs_traffic.err
  run $NCU --set full --clock-control none --import-source on -k regex:dcgs_update_kernel -s 20 -c 1 \
      -o $O/dcgs_update_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_dcgs.log 2>&1
  run $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiApply \
      -s 2 -c 1 -o $O/apply_full python scripts/perf_ops.py --reps 1 > $O/ncu_apply.log 2>&1
fi
