mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_c5.jsonl 2> gpurun_out/final_c5.err
for c in c1 c2 c3 c4 img32 img64 img128 img256 img512; do python bench.py --config $c >> gpurun_out/final_all.jsonl 2>> gpurun_out/final_all.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c5.csv python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/final_ncu_bench.log 2>&1; tail -1 gpurun_out/final_ncu_bench.log
ncu --set full --clock-control none --import-source on -k regex:"spread3_tmapad|interp3" -c 2 -o gpurun_out/final_kern python tools/profile_apply.py --config c5 --reps 1 > gpurun_out/final_ncu_kern.log 2>&1; tail -1 gpurun_out/final_ncu_kern.log
