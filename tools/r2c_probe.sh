# 32-node spread shape for c5; interp source-level profile; c2 launch list
mkdir -p gpurun_out
python tools/profile_apply.py --config c5 --reps 3 --per-dir 2>&1 | grep dir > gpurun_out/r2c_shape.log; cat gpurun_out/r2c_shape.log
python bench.py > gpurun_out/r2c_c5.jsonl 2> gpurun_out/r2c_c5.err; tail -c 200 gpurun_out/r2c_c5.jsonl
ncu --set full --clock-control none --import-source on -k regex:"interp3" -c 2 -o gpurun_out/r2c_interp python tools/profile_apply.py --config c5 --reps 1 > gpurun_out/r2c_ncu.log 2>&1; tail -1 gpurun_out/r2c_ncu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_c2_launches.csv python tools/profile_apply.py --config c2 --reps 3 > gpurun_out/r2c_c2ncu.log 2>&1; tail -1 gpurun_out/r2c_c2ncu.log
