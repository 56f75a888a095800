#!/bin/bash
# one gpurun payload: debug script, gpu tests, smoke
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python ${DEBUG_SCRIPT:-tools/debug_small.py} > gpurun_out/debug.log 2>&1; echo EXIT $? >> gpurun_out/debug.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_X} ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
