mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "divergence_parity_subsample or deterministic_spread_is" 2>&1 | grep -E "passed|failed|assert np" | head -3; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_protocol.py -m gpu -q -x -k "variants or occupancies or gridding or deterministic or c5 or c3 or box or emulated or nccl or divergence" > gpurun_out/pipe_pytest.log 2>&1; tail -2 gpurun_out/pipe_pytest.log
for c in c5 c3; do for v in "SK_X=0" "SK_SPREAD3_NOPIPE=1"; do echo "$c $v"; env $v python tools/profile_apply.py --config $c --reps 3 --per-dir 2>&1 | grep dir; done; done > gpurun_out/pipe_ab.log 2>&1; cat gpurun_out/pipe_ab.log
