# stage times of the small workloads (c2, img256, c1) with the library's CUDA-event profiler, and
# the bench step rate
for c in c2 img256; do echo "== $c"; python tools/profile_apply.py --config $c --reps 10 2>&1 | grep -v "^plan"; done
SK_BENCH_STAGE_PROFILE=0 python bench.py --config c2 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 bench it/s', d['value'], 'ms/step', d['ms_per_step'], 'launches/step', d['gpu_launches']/d['steps'])"
SK_DETERMINISTIC=0 SK_BENCH_STAGE_PROFILE=0 python bench.py --config c2 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2 (atomics) bench it/s', d['value'], 'ms/step', d['ms_per_step'])"
