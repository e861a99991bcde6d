# spread item floor (SK_SPREAD_ITEM_MIN) against the spread time, deterministic and atomic modes
for c in img512 c2 img64 c4 c3; do for det in 1 0; do for im in 64 128 256 512; do
  printf "%s det=%s item_min=%s " $c $det $im
  SK_DETERMINISTIC=$det SK_SPREAD_ITEM_MIN=$im python tools/profile_apply.py --config $c --reps 10 2>&1 | grep spread
done; done; done
