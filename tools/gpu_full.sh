#!/bin/bash
# gpurun payload: gpu tests, smoke, bench (ours + reference arm), ncu launch
# list of one full c4 solve, ncu --set full of the hot kernels (summarised on
# the box, the .ncu-rep files stay in /tmp to respect the copy-back limit)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo EXIT $? >> gpurun_out/bench.log
  if [ -n "$REF" ]; then
    timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo EXIT $? >> gpurun_out/bench_ref.log
  fi
fi
if [ -z "$SKIP_NCU" ]; then
  CFG=${CFG:-c4}
  timeout 300 python tools/solve_once.py --config $CFG > gpurun_out/plain.log 2>&1 || exit 0
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python tools/solve_once.py --config $CFG > gpurun_out/ncu_list.log 2>&1
  python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_$CFG.txt 2>&1
  for K in ${KERNELS:-k_combine k_apply_gram}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 -o /tmp/prof_$K -f python tools/solve_once.py --config $CFG --max-m 40 > gpurun_out/ncu_$K.log 2>&1
    python tools/ncu_summary.py /tmp/prof_$K.ncu-rep gpurun_out/prof_${K}_${CFG}.json > /dev/null 2>&1
    ncu -i /tmp/prof_$K.ncu-rep --page source --csv > gpurun_out/prof_${K}_sass.csv 2>/dev/null
  done
fi
