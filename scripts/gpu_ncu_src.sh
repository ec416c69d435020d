# ncu --set full with source-level stall sampling of the decode gate_up GEMM (one launch)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 6 -c 1 -o gpurun_out/prof_src python scripts/prof_gemm.py ${SHAPE:-16 22016 4096} 8 > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_src.log
