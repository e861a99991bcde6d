# final validation of HEAD: GPU suite, smoke, driver bench command, ncu launch list, ncu of both kernels
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=5 > gpurun_out/fin2_pytest.log 2>&1; tail -2 gpurun_out/fin2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; tail -1 gpurun_out/fin2_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin2_c5.jsonl 2> gpurun_out/fin2_c5.err; tail -c 200 gpurun_out/fin2_c5.jsonl; echo
for c in c2 c3 c4 img64; do python bench.py --config $c --no-cpu-baseline >> gpurun_out/fin2_all.jsonl 2>/dev/null; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin2_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/fin2_ncu.log 2>&1; echo ncu_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"spread3_t28|interp3" -c 6 -o gpurun_out/fin2_kern python tools/profile_apply.py --config c5 --reps 1 --per-dir > gpurun_out/fin2_ncu_kern.log 2>&1; tail -1 gpurun_out/fin2_ncu_kern.log
