mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "r1 or emulated or nccl" > gpurun_out/r1mr_pytest.log 2>&1; tail -3 gpurun_out/r1mr_pytest.log
