for c in 5 4 2; do
  for bv in 0 1 2 3 4 5; do HANF_BV=$bv python scripts/policy_sweep.py $c "" 2>&1 | tail -1 | sed "s/^/bv$bv /"; done
done
