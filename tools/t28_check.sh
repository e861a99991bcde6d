mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or occupancies or gridding or deterministic or matvec_parity_full or box_exchange" > gpurun_out/t28_pytest.log 2>&1; tail -3 gpurun_out/t28_pytest.log
bash tools/ab_lib.sh old28 c5 c3 > gpurun_out/t28_ab.log 2>&1; cat gpurun_out/t28_ab.log
