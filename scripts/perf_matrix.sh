# Perf experiments: per-class times of one apply + one V-cycle under RTE_TC_DBG switches ($DBGS),
# then role counters for the level-0 conv ($ROLES).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for d in ${DBGS:-0 128}; do
  echo -n "dbg=$d "; RTE_TC_DBG=$d timeout 120 python scripts/perf_ops.py 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in j.items() if k.startswith('conv3x3_tc') or k.startswith('apply') or k.startswith('conv1x1_tc@512x32') or k.startswith('_total')})"
done
for d in ${ROLES:-73792}; do echo "== roles dbg=$d"; RTE_LIB_PATH=${PROF_LIB:-var_libs/librte_prof.so} RTE_TC_DBG=$d timeout 120 python scripts/perf_roles.py 2>&1 | tail -24; done
