cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
for m in ${MODES:-0 1 2 3}; do echo "=== FIREQ_DEBUG_MODE=$m"; FIREQ_DEBUG_MODE=$m timeout 300 python scripts/trace_gemm.py 2>&1 | grep -E "M=16 N=22016" -A 14 | grep -E "first_data|mma_done|cyc" ; done
