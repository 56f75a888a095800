#!/bin/bash
# gpurun payload: gpu tests, c4 bench, full-solve launch list summary
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} ${BENCH_ARGS} > gpurun_out/bench_c4.log 2>&1; echo EXIT $? >> gpurun_out/bench_c4.log
fi
if [ -z "$SKIP_LIST" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python tools/solve_once.py --config ${CFG:-c4} > gpurun_out/ncu_list.log 2>&1
  python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launch_summary_${CFG:-c4}.txt 2>&1
fi
