#!/bin/bash
# A/B of environment switches (bench c4, no e2e): ENVS="A=1 B=1" one per run, "base" = none
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for e in ${ENVS:-base}; do
  if [ "$e" = base ]; then timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_env_base.log 2>&1;
  else env $e timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_env_${e%%=*}.log 2>&1; fi
done
