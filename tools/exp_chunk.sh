#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for g in 32 64 96; do
  KRY_PASS2_CHUNK=$g timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_chunk_$g.log 2>&1
done
