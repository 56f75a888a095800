#!/bin/bash
# quick GPU iteration: small-case correctness (fused vs 2-kernel) + c4 bench line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/fused_probe.py ${PROBE_CFGS:-c2} > gpurun_out/fused_probe.log 2>&1; echo EXIT $? >> gpurun_out/fused_probe.log
timeout 600 python bench.py --steps ${STEPS:-2} --warmup ${WARMUP:-1} --no-cpu-baseline ${BENCH_ARGS:---no-e2e} > gpurun_out/bench_quick.log 2>&1; echo EXIT $? >> gpurun_out/bench_quick.log
