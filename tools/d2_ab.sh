# d = 2: y taps in the kernel (default) vs from the table (SK_D2_TAPS_TABLE=1)
for c in c4 c2 img512; do for t in 0 1; do
  printf "%s table=%s " $c $t; SK_D2_TAPS_TABLE=$t python tools/profile_apply.py --config $c --reps 10 --per-dir 2>&1 | grep dir | tr '\n' ' '; echo
done; done
