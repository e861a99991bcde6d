# programmatic dependent launch on the d = 2 chain: parity, then bench A/B (SK_NO_PDL)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fftconv2 or image or c2 or deterministic or random_configs or trace or graph or enonpos" > gpurun_out/pdl_pytest.log 2>&1; tail -2 gpurun_out/pdl_pytest.log
for c in c2 img64 img512; do python bench.py --config $c --no-cpu-baseline; SK_NO_PDL=1 python bench.py --config $c --no-cpu-baseline; done > gpurun_out/pdl_bench.jsonl 2> gpurun_out/pdl_bench.err
python - <<'PY'
import json
for l in open("gpurun_out/pdl_bench.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["workload"], round(d["value"],1), round(d["e2e"]["value"],1))
PY
