#!/bin/bash
# gpurun payload: gpu tests, c4 bench, full ncu capture of both hot kernels
# (the .ncu-rep files are summarised on the box: raw + source CSV, then removed,
# to stay under the 64 MiB copy-back limit)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
fi
timeout 1200 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} > gpurun_out/bench_c4.log 2>&1; echo EXIT $? >> gpurun_out/bench_c4.log
if [ -z "$SKIP_NCU" ]; then
  timeout 300 python tools/solve_once.py --config c4 --max-m 40 > gpurun_out/plain.log 2>&1 || exit 0
  for K in ${KERNELS:-k_combine k_apply_gram}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 -o /tmp/prof_$K -f python tools/solve_once.py --config c4 --max-m 40 > gpurun_out/ncu_$K.log 2>&1
    ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/prof_${K}_raw.csv 2>/dev/null
    ncu -i /tmp/prof_$K.ncu-rep --page source --csv > gpurun_out/prof_${K}_sass.csv 2>/dev/null
  done
fi
