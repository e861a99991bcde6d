# A/B of an alternative build (paper_2201_07524_b200/lib/$1.so) against the default library
ALT=$1; shift
for i in 1 2; do for c in "$@"; do
  printf "%s default " $c; python tools/profile_apply.py --config $c --reps 4 --per-dir 2>&1 | grep dir | tr '\n' ' '; echo
  printf "%s %s " $c $ALT; SK_LIB_PATH=$PWD/paper_2201_07524_b200/lib/$ALT.so python tools/profile_apply.py --config $c --reps 4 --per-dir 2>&1 | grep dir | tr '\n' ' '; echo
done; done
