for r in 1 2 3; do for dv in 1776 4736; do printf "c4 div=%s " $dv; SK_SPREAD_ITEM_DIV=$dv python tools/profile_apply.py --config c4 --reps 10 2>&1 | grep spread; done; done
for dv in 1776 4736; do printf "img256 div=%s " $dv; SK_SPREAD_ITEM_DIV=$dv python tools/profile_apply.py --config img256 --reps 10 2>&1 | grep spread; done
