set -x
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/r02_ref_c5.json 2> gpurun_out/r02_ref_c5.err; echo ref rc=$?
python scripts/hot_fraction.py 5 > gpurun_out/r02_hot5.txt 2>&1
python scripts/hot_fraction.py 4 > gpurun_out/r02_hot4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_kernel -c 1 -f -o gpurun_out/r02_c5_full python scripts/one_step_rmat.py 28 1 > gpurun_out/r02_c5_ncu.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-config2 > gpurun_out/r02_c5_launch.log 2>&1; echo ncu2 rc=$?
