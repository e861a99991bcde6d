mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/v1_pytest.log 2>&1; tail -3 gpurun_out/v1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1; tail -2 gpurun_out/v1_smoke.log
python bench.py > gpurun_out/v1_c5.jsonl 2> gpurun_out/v1_c5.err; tail -c 400 gpurun_out/v1_c5.jsonl
for c in c1 c2 c3 c4 c1r1; do python bench.py --config $c --no-cpu-baseline >> gpurun_out/v1_all.jsonl 2>> gpurun_out/v1_all.err; done
