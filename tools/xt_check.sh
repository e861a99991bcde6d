mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or occupancies or gridding or c5 or c3 or divergence_parity" > gpurun_out/py_pytest.log 2>&1; tail -2 gpurun_out/py_pytest.log
bash tools/ab_lib.sh py_old c5 c3 > gpurun_out/py_ab.log 2>&1; cat gpurun_out/py_ab.log
