#!/bin/bash
# gpurun payload: full ncu captures of the eigen-engine kernels late in a c4 solve
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/solve_once.py --config c4 > gpurun_out/plain.log 2>&1 || exit 0
for spec in k_eig_secular:1600 k_eig_zhat:1600 k_eig_vec_partial:1600 k_eig_vec_finish:1600 k_eig_deflate:1600 k_cauchy:200; do
  K=${spec%%:*}; S=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/prof_$K -f python tools/solve_once.py --config c4 > gpurun_out/ncu_$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/prof_${K}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page source --csv > gpurun_out/prof_${K}_sass.csv 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page details > gpurun_out/prof_${K}_details.txt 2>/dev/null
done
