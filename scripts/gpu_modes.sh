cd $GRAFT_REPO_ROOT
for m in 0 1 2 3 4 5 6; do echo "dbg=$m"; FIREQ_DEBUG_MODE=$m timeout 60 python scripts/time_gemm.py 16 22016 4096 16 4096 11008; done > gpurun_out/modes.txt 2>&1
for m in 0 1 2; do FIREQ_DEBUG_MODE=$m ROT=1 timeout 60 python scripts/evt_gemm.py; done > gpurun_out/evt_modes.txt 2>&1
cat gpurun_out/modes.txt; cat gpurun_out/evt_modes.txt
