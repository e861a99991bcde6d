# three back-to-back default bench runs (reproducibility of the c5 line)
mkdir -p gpurun_out
for i in 1 2 3; do python bench.py --no-cpu-baseline >> gpurun_out/repro_c5.jsonl 2>> gpurun_out/repro_c5.err; done
