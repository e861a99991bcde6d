mkdir -p gpurun_out
bash tools/ab_env.sh "c2 c3 img64" "SK_X=0" "SK_NO_PDL=1" 3 > gpurun_out/r2e_pdl.log 2>&1; cat gpurun_out/r2e_pdl.log
bash tools/ab_env.sh "c3" "SK_X=0" "SK_NO_XPAIRS=1" 3 > gpurun_out/r2e_xp.log 2>&1; cat gpurun_out/r2e_xp.log
