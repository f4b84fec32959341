set -x
python scripts/policy_sweep.py 5 ";HANF_GATHER=50,HANF_HOT_MB=32;HANF_GATHER=50,HANF_HOT_MB=48;HANF_GATHER=50,HANF_HOT_MB=64;HANF_GATHER=50,HANF_HOT_MB=80;HANF_GATHER=50,HANF_HOT_MB=100;HANF_GATHER=51,HANF_HOT_MB=64" > gpurun_out/r02_pol5.txt 2>&1
python scripts/policy_sweep.py 4 ";HANF_GATHER=50,HANF_HOT_MB=32;HANF_GATHER=50,HANF_HOT_MB=64;HANF_GATHER=50,HANF_HOT_MB=96;HANF_GATHER=51,HANF_HOT_MB=64" > gpurun_out/r02_pol4.txt 2>&1
python scripts/policy_sweep.py 2 ";HANF_GATHER=50,HANF_HOT_MB=64,HANF_RELABEL=1;HANF_RELABEL=1" > gpurun_out/r02_pol2.txt 2>&1
cat gpurun_out/r02_pol5.txt gpurun_out/r02_pol4.txt gpurun_out/r02_pol2.txt
