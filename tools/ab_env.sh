# A/B of environment switches on bench lines: ab_env.sh "<cfgs>" "<env A>" "<env B>" [reps]
CFGS=$1; A=$2; B=$3; R=${4:-2}
for r in $(seq $R); do for c in $CFGS; do for v in "$A" "$B"; do
  val=$(env $v SK_BENCH_STAGE_PROFILE=0 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "$c [$v] $val"
done; done; done
