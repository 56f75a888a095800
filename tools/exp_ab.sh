#!/bin/bash
# A/B of experimental library builds in exp/lib_<name>.so (bench c4, no e2e)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in ${VARIANTS:-base contig}; do
  KRY_LIB_PATH=$PWD/exp/lib_$v.so timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_$v.log 2>&1
done
