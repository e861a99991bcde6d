# cost of the spread's per-cell region update and of the global region flush (timing-only builds)
for c in c3 c5; do for lib in libsk_nfft libsk_t_CELL libsk_t_REGION; do for det in 1 0; do
  printf "%s %s det=%s " $c $lib $det
  SK_DETERMINISTIC=$det SK_LIB_PATH=$PWD/paper_2201_07524_b200/lib/$lib.so python tools/profile_apply.py --config $c --reps 4 --per-dir 2>&1 | grep "dir" | tr '\n' ' '; echo
done; done; done
