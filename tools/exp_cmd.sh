cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset KRY_LIB_PATH; else export KRY_LIB_PATH=exp/$v/libkrymat_b200.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_combine|k_apply_gram" -c 120 --csv --log-file /tmp/l_$v.csv python tools/solve_once.py --config c4 --max-m 60 > gpurun_out/exp_$v.log 2>&1
  python tools/launch_summary.py /tmp/l_$v.csv > gpurun_out/exp_sum_$v.txt
done
