# ncu evidence of this round's union kernels (run on the GPU box)
set -x
ncu --set full --clock-control none --import-source on -k regex:union_kernel -c 1 \
    -o gpurun_out/r02b_config2_full -f python scripts/policy_sweep.py 2 "" > gpurun_out/r02b_ncu2.log 2>&1
ncu -i gpurun_out/r02b_config2_full.ncu-rep --page raw --csv > gpurun_out/r02b_config2_full.csv
ncu --set full --clock-control none --import-source on -k regex:union_kernel -c 1 \
    -o gpurun_out/r02b_config5_full -f python scripts/policy_sweep.py 5 "" > gpurun_out/r02b_ncu5.log 2>&1
ncu -i gpurun_out/r02b_config5_full.ncu-rep --page raw --csv > gpurun_out/r02b_config5_full.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02b_launches5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-e2e --no-config2 > gpurun_out/r02b_l5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02b_launches2.csv python bench.py --config 2 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/r02b_l2.log 2>&1
ls -la gpurun_out/
