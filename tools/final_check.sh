# round-end checkpoint: GPU suite, smoke, the driver's bench command, the reference arm, all
# workloads, the ncu launch list of the bench command
set -x
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_c5.jsonl 2> gpurun_out/final_bench_c5.err; tail -c 300 gpurun_out/final_bench_c5.jsonl
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.jsonl 2>&1; tail -c 300 gpurun_out/final_bench_ref.jsonl
bash tools/bench_all.sh > gpurun_out/final_bench_all.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1; echo ncu_rc=$?
