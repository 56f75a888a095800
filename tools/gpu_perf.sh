#!/bin/bash
# gpurun payload: tests, bench, ncu launch list + full capture of one kernel
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CFG=${CFG:-c4}
MAXM=${MAXM:-40}
KREGEX=${KREGEX:-k_combine}
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py --config $CFG --steps ${STEPS:-2} --warmup ${WARMUP:-1} ${BENCH_ARGS} > gpurun_out/bench_$CFG.log 2>&1; echo EXIT $? >> gpurun_out/bench_$CFG.log
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 300 python tools/solve_once.py --config $CFG --max-m $MAXM > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${NCU_SKIP:-600} -c ${NCU_COUNT:-400} --csv --log-file gpurun_out/launches_$CFG.csv python tools/solve_once.py --config $CFG --max-m $MAXM > gpurun_out/ncu_list.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${NCU_KSKIP:-5} -c 1 -o gpurun_out/prof_${KREGEX} -f python tools/solve_once.py --config $CFG --max-m $MAXM > gpurun_out/ncu_full.log 2>&1
  echo EXIT $? >> gpurun_out/ncu_full.log
fi
