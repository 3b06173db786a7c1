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
  R=/tmp/rte_ncu_r02   # .ncu-rep files stay on the box (gpurun_out/ is capped at 64 MiB); their summaries travel
  mkdir -p $R
  run timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
  python scripts/summarize_ncu.py launches $O/launches.csv > $O/launches_summary.txt
  run timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"cgs_kernel|dcgs_update_kernel" --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      > $O/cgs_traffic.csv 2> $O/cgs_traffic.err
  run timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dcgs_update_kernel -s 20 -c 1 \
      -f -o $R/dcgs_update_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_dcgs.log 2>&1
  python scripts/summarize_ncu.py full $R/dcgs_update_full.ncu-rep > $O/dcgs_update_full.txt
  run timeout 600 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiApply \
      -s 2 -c 1 -f -o $R/apply_full python scripts/perf_ops.py --reps 1 > $O/ncu_apply.log 2>&1
  python scripts/summarize_ncu.py full $R/apply_full.ncu-rep > $O/apply_tma_full.txt
  # one whole round of tensor-core GEMM launches (the apply and every conv of one V-cycle, in launch order)
  run timeout 1200 $NCU --set full --clock-control none --kernel-name-base demangled -k regex:gemm3xtf32 \
      -s 120 -c 61 -f -o $R/vcycle_gemms_full python scripts/perf_ops.py --reps 1 > $O/ncu_vcycle.log 2>&1
  python scripts/summarize_ncu.py full $R/vcycle_gemms_full.ncu-rep > $O/vcycle_gemms_full.txt
  rm -f $O/launches.csv.tmp
fi
