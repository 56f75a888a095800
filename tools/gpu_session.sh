#!/bin/bash
# gpurun payload for measurement sessions.  Steps are selected by env vars:
#   PEAK=1      fp64 DFMA/DMMA/reciprocal peak microbenchmark -> gpurun_out/fp64_peak.json
#   TESTS=1     pytest -m gpu (PYTEST_K filters)      -> gpurun_out/gpu_tests.log
#   HIST="c3 c5" histories through the API              -> gpurun_out/hist_*.npz
#   BENCH="args" python bench.py args                    -> gpurun_out/bench.log
#   NCU="cfg:kernel_regex:skip ..." ncu --set full of one launch each
#   LIST=cfg    ncu launch list of one solve             -> gpurun_out/launches_cfg.txt
#   CMD="..."   any extra command (output in gpurun_out/cmd.log)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log 2>&1
if [ -n "$PEAK" ]; then
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu > gpurun_out/fp64_peak.log 2>&1
  timeout 120 /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>> gpurun_out/fp64_peak.log
fi
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
fi
if [ -n "$HIST" ]; then
  timeout 900 python tools/dump_histories.py $HIST > gpurun_out/hist.log 2>&1; echo EXIT $? >> gpurun_out/hist.log
fi
if [ -n "$BENCH" ]; then
  timeout 1200 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo EXIT $? >> gpurun_out/bench.log
fi
if [ -n "$CMD" ]; then
  timeout 1500 bash -c "$CMD" > gpurun_out/cmd.log 2>&1; echo EXIT $? >> gpurun_out/cmd.log
fi
if [ -n "$LIST" ]; then
  timeout 300 python tools/solve_once.py --config $LIST > gpurun_out/plain_$LIST.log 2>&1
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python tools/solve_once.py --config $LIST > gpurun_out/ncu_list_$LIST.log 2>&1
  python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_$LIST.txt 2>&1
fi
for spec in $NCU; do
  IFS=: read CFG K SKIP MAXM <<< "$spec"
  tag=${K}_${CFG}_s${SKIP}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/prof_$tag -f python tools/solve_once.py --config $CFG ${MAXM:+--max-m $MAXM} > gpurun_out/ncu_$tag.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$tag.ncu-rep gpurun_out/prof_$tag.json > /dev/null 2>&1
done
exit 0
