# A/B of the round-1 library against the current one on c5 applies (profile_apply stage times)
for i in 1 2; do
echo "== r1 lib"; SK_LIB_PATH=$PWD/paper_2201_07524_b200/lib/libsk_nfft_r1.so python tools/profile_apply.py --config c5 --reps 4 2>&1 | grep -E "spread|interp"
echo "== current det=0"; SK_DETERMINISTIC=0 python tools/profile_apply.py --config c5 --reps 4 2>&1 | grep -E "spread|interp"
echo "== current det=1"; python tools/profile_apply.py --config c5 --reps 4 2>&1 | grep -E "spread|interp"
done
