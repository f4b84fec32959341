python -c "
from cuda.bindings import runtime as rt
print('max persisting', rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0))
print('l2', rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0))
" 2>&1 | tail -3
python scripts/policy_sweep.py 5 ";HANF_GATHER=50,HANF_HOT_MB=32,HANF_L2_PERSIST_MB=48;HANF_GATHER=50,HANF_HOT_MB=48,HANF_L2_PERSIST_MB=64;HANF_GATHER=50,HANF_HOT_MB=64,HANF_L2_PERSIST_MB=80;HANF_GATHER=50,HANF_HOT_MB=80,HANF_L2_PERSIST_MB=100;HANF_GATHER=50,HANF_HOT_MB=96,HANF_L2_PERSIST_MB=120" 2>&1 | grep union
HANF_PROFILE=1 HANF_GATHER=50 HANF_HOT_MB=64 HANF_L2_PERSIST_MB=80 timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:union_kernel -c 1 python scripts/one_step_rmat.py 28 1 2>&1 | grep -E "dram__|lts__|gpu__time|set-aside"
