# dev aid: L2 access-policy window effect on config 5 (sweep, estimate_nf) and config 2 after it
python scripts/policy_sweep.py 5 ";HANF_L2_WINDOW_MB=0" 2>&1 | tail -2
python scripts/policy_sweep.py 2 "" 2>&1 | tail -1
python scripts/e2e_breakdown5.py 2>&1 | grep -E "^create"
HANF_L2_WINDOW_MB=0 python scripts/e2e_breakdown5.py 2>&1 | grep -E "^create" | sed "s/^/nowin /"
