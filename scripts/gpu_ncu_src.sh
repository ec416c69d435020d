# fine-grained warp-stall sampling of one GEMM launch (source page)
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 > /dev/null
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_w4a8_gemm -s 2 -c 1 -o gpurun_out/${NCU_NAME:-src} python scripts/prof_gemm.py ${NCU_SHAPE:-16 22016 4096} 4 > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_src.log
