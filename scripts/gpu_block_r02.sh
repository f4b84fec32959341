# round-2 (session 4) evidence for the source-blocked dense sweeps
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02k_gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02k_gputest.log
HANF_LIB=checked timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02k_gputest_checked.log 2>&1; echo "checked tests rc=$?"; tail -2 gpurun_out/r02k_gputest_checked.log
(time python bench.py) > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo "bench rc=$?"; tail -4 gpurun_out/r02k_bench.err
(time python bench.py --impl reference) > gpurun_out/r02k_ref.json 2> gpurun_out/r02k_ref.err; echo "ref rc=$?"; tail -4 gpurun_out/r02k_ref.err
ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 2 -c 2 \
    -o gpurun_out/r02k_config5_full -f python scripts/block_time.py 5 "HANF_BLOCK=1" > gpurun_out/r02k_ncu5.log 2>&1
ncu -i gpurun_out/r02k_config5_full.ncu-rep --page raw --csv > gpurun_out/r02k_config5_full.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/r02k_launches5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-e2e --no-config2 > gpurun_out/r02k_l5.log 2>&1
echo done
