for c in c5 c3 c4 c2; do for d in 0 1; do echo "== $c det=$d"; SK_DETERMINISTIC=$d python tools/profile_apply.py --config $c --reps 3 2>&1 | grep -E "spread|interp"; done; done
