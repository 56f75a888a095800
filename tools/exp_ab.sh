#!/bin/bash
# A/B of experimental library builds in exp/lib_<name>.so (bench c4, no e2e)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in ${VARIANTS:-base contig}; do
  KRY_LIB_PATH=$PWD/exp/lib_$v.so timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_$v.log 2>&1
done
if [ -n "$EIG_LIST" ]; then
  for v in ${VARIANTS:-base}; do
    KRY_LIB_PATH=$PWD/exp/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_eig_secular --csv --log-file /tmp/eig_$v.csv python tools/solve_once.py --config c4 > /dev/null 2>&1
    python tools/launch_summary.py /tmp/eig_$v.csv > gpurun_out/eig_$v.txt 2>&1
  done
fi
