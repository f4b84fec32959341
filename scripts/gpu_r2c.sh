# round-2 batch: GPU tests, bench (config 5) + reference arm, e2e breakdown,
# ncu of the current config-3/4 union kernels, compute-sanitizer
set -x
python -m pytest tests -q -m gpu -x --timeout 3000 > gpurun_out/r02_gputests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r02_gputests.log
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo bench rc=$?
python scripts/e2e_breakdown5.py > gpurun_out/r02_e2e5.log 2>&1
for c in 4 3; do
  timeout 900 ncu --set full --clock-control none -k regex:union_kernel -c 1 -f -o /tmp/r02_c${c}_full python scripts/policy_sweep.py $c "" > gpurun_out/r02_c${c}_ncu.log 2>&1
  ncu -i /tmp/r02_c${c}_full.ncu-rep --page raw --csv > gpurun_out/r02_c${c}_full_raw.csv 2>&1
done
