# 28-tile spread: bench line, 32-node shape A/B, ncu of the new kernel, small-workload stages
mkdir -p gpurun_out
python bench.py > gpurun_out/r2b_c5.jsonl 2> gpurun_out/r2b_c5.err; tail -c 300 gpurun_out/r2b_c5.jsonl
for v in 0 1000000000; do echo "SEG_DENSE_MIN=$v"; SK_SEG_DENSE_MIN=$v python tools/profile_apply.py --config c5 --reps 3 --per-dir 2>&1 | grep dir; done > gpurun_out/r2b_shape.log 2>&1; cat gpurun_out/r2b_shape.log
bash tools/small_profile.sh > gpurun_out/r2b_small.log 2>&1; cat gpurun_out/r2b_small.log
ncu --set full --clock-control none --import-source on -k regex:"spread3_tmapad" -c 2 -o gpurun_out/r2b_spread python tools/profile_apply.py --config c5 --reps 1 > gpurun_out/r2b_ncu.log 2>&1; tail -2 gpurun_out/r2b_ncu.log
