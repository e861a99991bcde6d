# spread work-item size divisor (SK_SPREAD_ITEM_DIV: item nodes = count / div, floor 64, cap 4096)
for c in c5 c4 c3 c2 img512; do for dv in 1776 4736; do
  printf "%s div=%s " $c $dv; SK_SPREAD_ITEM_DIV=$dv python tools/profile_apply.py --config $c --reps 6 2>&1 | grep spread
done; done
