#!/usr/bin/env bash
# Turnkey 1 -> 8 GPU scaling run of the c5 workload (BASELINE.json configs[4]) on one node:
# one rank per GPU over NCCL, the exact launch the driver uses. Writes one JSON line per N to
# profiles/scaling_<tag>.jsonl and the NCCL init lines (ranks, channels, NVLS) to
# profiles/scaling_<tag>_nccl.log. Expected per-N it/s from the DESIGN.md §7 model (measured 1-GPU
# stages, box all-reduce, redundant pruned FFT): N=1 17.0, N=2 ~33, N=4 ~64, N=8 ~120 (~7x).
#
#   bash tools/run_scaling.sh [tag] [steps] [warmup]
set -euo pipefail
cd "$(dirname "$0")/.."
TAG=${1:-r2}
STEPS=${2:-3}
WARMUP=${3:-3}
NGPU=$(nvidia-smi -L | wc -l)
OUT=profiles/scaling_${TAG}.jsonl
LOG=profiles/scaling_${TAG}_nccl.log
: > "$OUT"
: > "$LOG"
for N in 1 2 4 8; do
  if [ "$N" -gt "$NGPU" ]; then echo "skip N=$N (only $NGPU GPUs)"; continue; fi
  if [ "$N" -eq 1 ]; then
    python bench.py --gpus 1 --steps "$STEPS" --warmup "$WARMUP" 2>>"$LOG" | tail -1 >> "$OUT"
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus "$N" --steps "$STEPS" --warmup "$WARMUP" \
      2>>"$LOG" | tail -1 >> "$OUT"
  fi
  python - "$OUT" <<'EOF'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
r = rows[-1]
base = rows[0]["value"]
print(f"N={r['n_gpus']}: {r['value']:.2f} it/s  ({r['value'] / base:.2f}x of N=1)  e2e {r.get('e2e', {}).get('value')}")
EOF
done
grep -E "NCCL INFO (comm|NVLS|Channel 00)" "$LOG" | head -40 || true
