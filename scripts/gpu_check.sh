#!/bin/bash
# GPU pass: parity tests (fail fast), bench, ncu launch list + full capture of a kernel regex ($1).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
KREGEX="${1:-gemm3xtf32}"
TESTS="${TESTS:-tests}"
timeout 1500 python -m pytest $TESTS -m gpu -q ${PYX--x} -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
PT=$?
echo "pytest exit $PT" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
if [ $PT -ne 0 ] && [ -z "$FORCE" ]; then echo "tests failed: skipping bench/ncu"; exit 1; fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
BE=$?
echo "bench exit $BE" >> gpurun_out/bench.err
[ $BE -ne 0 ] && { tail -20 gpurun_out/bench.err; exit 1; }
cat gpurun_out/bench.json | head -c 600; echo
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
     --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu1 exit $?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 40 -c 3 \
     -o gpurun_out/prof_top $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
