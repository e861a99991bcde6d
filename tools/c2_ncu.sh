mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"spread2|interp2|fc2_" -c 10 -o gpurun_out/c2_kern python tools/profile_apply.py --config c2 --reps 2 > gpurun_out/c2_ncu.log 2>&1; tail -1 gpurun_out/c2_ncu.log
python /root/repo/tools/microbench_run.py 2>/dev/null || (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb tools/microbench.cu && /tmp/mb > gpurun_out/microbench_r2.txt 2>&1; grep -i "t28\|spread mix m16" gpurun_out/microbench_r2.txt)
