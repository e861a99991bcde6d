for v in "SK_X=0" "SK_SEG_DENSE_MIN=200" "SK_SEG_DENSE_MIN=1000"; do echo "c5 $v"; env $v python tools/profile_apply.py --config c5 --reps 3 --per-dir 2>&1 | grep dir; done
