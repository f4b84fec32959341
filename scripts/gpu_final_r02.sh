# round-2 evidence: GPU tests, bench line, ncu of the current union kernels
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_gputest.log
python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"
ncu --set full --clock-control none --import-source on -k regex:union_kernel -c 1 \
    -o gpurun_out/r02d_config5_full -f python scripts/policy_sweep.py 5 "" > gpurun_out/r02d_ncu5.log 2>&1
ncu -i gpurun_out/r02d_config5_full.ncu-rep --page raw --csv > gpurun_out/r02d_config5_full.csv
ncu --set full --clock-control none --import-source on -k regex:union_kernel -c 1 \
    -o gpurun_out/r02d_config2_full -f python scripts/policy_sweep.py 2 "" > gpurun_out/r02d_ncu2.log 2>&1
ncu -i gpurun_out/r02d_config2_full.ncu-rep --page raw --csv > gpurun_out/r02d_config2_full.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/r02d_launches5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-e2e --no-config2 > gpurun_out/r02d_l5.log 2>&1
echo done
