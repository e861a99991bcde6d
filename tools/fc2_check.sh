# d = 2 shared-memory FFT convolution: parity, then stage times and bench lines of the d = 2 workloads
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fftconv2" > gpurun_out/fc2_pytest.log 2>&1; tail -3 gpurun_out/fc2_pytest.log
python -m pytest tests -m gpu -q -x > gpurun_out/fc2_pytest_all.log 2>&1; tail -3 gpurun_out/fc2_pytest_all.log
for c in c2 img64 img512; do echo "== $c"; python tools/profile_apply.py --config $c --reps 10 2>&1 | grep -v "^plan"; echo "-- cufft"; SK_NO_FFTCONV2=1 python tools/profile_apply.py --config c2 --reps 10 2>&1 | grep -v "^plan"; done > gpurun_out/fc2_stages.log 2>&1
for c in c2 c4 img64 img256 img512; do python bench.py --config $c --no-cpu-baseline; SK_NO_FFTCONV2=1 python bench.py --config $c --no-cpu-baseline; done > gpurun_out/fc2_bench.jsonl 2> gpurun_out/fc2_bench.err
python - <<'PY'
import json
for l in open("gpurun_out/fc2_bench.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["workload"], round(d["value"],1), d["e2e"]["value"])
PY
