# round-2 checkpoint: GPU suite, smoke, the driver's bench command, the reference arm, all
# workloads, the ncu launch list of the bench command, --set full of the two c5 kernels (both sides)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/fin_pytest.log 2>&1; tail -2 gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_c5.jsonl 2> gpurun_out/fin_c5.err; tail -c 200 gpurun_out/fin_c5.jsonl; echo
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.jsonl 2>&1; tail -c 200 gpurun_out/fin_ref.jsonl; echo
bash tools/bench_all.sh > gpurun_out/fin_all.jsonl 2>&1
SK_DETERMINISTIC=0 bash tools/bench_all.sh > gpurun_out/fin_all_atomic.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1; echo ncu_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"spread3_t28|interp3" -c 6 -o gpurun_out/fin_kern python tools/profile_apply.py --config c5 --reps 1 --per-dir > gpurun_out/fin_ncu_kern.log 2>&1; tail -1 gpurun_out/fin_ncu_kern.log
