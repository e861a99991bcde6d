# d = 3 PDL + 28-tile spread defaults: GPU suite, c3 x-pair A/B, c5 bench, ncu of both c5 spread launches
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1; tail -2 gpurun_out/r2d_pytest.log
for v in "" "SK_NO_XPAIRS=1"; do echo "c3 $v"; env $v python tools/profile_apply.py --config c3 --reps 5 --per-dir 2>&1 | grep dir; done > gpurun_out/r2d_c3xp.log 2>&1; cat gpurun_out/r2d_c3xp.log
python bench.py > gpurun_out/r2d_c5.jsonl 2> gpurun_out/r2d_c5.err; tail -c 250 gpurun_out/r2d_c5.jsonl; echo
python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2d_c3.jsonl 2>/dev/null; SK_NO_PDL=1 python bench.py --config c3 --no-cpu-baseline >> gpurun_out/r2d_c3.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/r2d_c3.jsonl'):
    d=json.loads(l); print('c3', d['value'])"
ncu --set full --clock-control none --import-source on -k regex:"spread3_tmapad" -c 2 -o gpurun_out/r2d_spread python tools/profile_apply.py --config c5 --reps 1 --per-dir > gpurun_out/r2d_ncu.log 2>&1; tail -1 gpurun_out/r2d_ncu.log
