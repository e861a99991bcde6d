# one bench line per workload (default steps; the small ones time ~1.5 s), for DESIGN.md §6b
for c in c1 c2 c3 c4 img64 img256 img512 c1r1; do
  python bench.py --config $c --warmup 3 2>/dev/null | tail -1
done
