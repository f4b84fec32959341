# round-2 measurement batch (config 5): bench, reference arm, ncu launch list
# and one --set full capture of the dense union kernel, exported to CSV here
# (the .ncu-rep itself is too big to travel back)
set -x
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/r02_ref_c5.json 2> gpurun_out/r02_ref_c5.err; echo ref rc=$?
timeout 900 ncu --set full --clock-control none -k regex:union_kernel -c 1 -f -o /tmp/r02_c5_full python scripts/one_step_rmat.py 28 1 > gpurun_out/r02_c5_ncu.log 2>&1; echo ncu rc=$?
ncu -i /tmp/r02_c5_full.ncu-rep --page raw --csv > gpurun_out/r02_c5_full_raw.csv 2>&1
ncu -i /tmp/r02_c5_full.ncu-rep --page details --csv > gpurun_out/r02_c5_full_details.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-config2 > gpurun_out/r02_c5_launch.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
