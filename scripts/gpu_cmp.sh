# A/B timing of decode GEMM shapes under FIREQ_DEBUG_MODE values given in $MODES
cd $GRAFT_REPO_ROOT
for m in ${MODES:-0}; do echo "== dbg=$m"; FIREQ_DEBUG_MODE=$m timeout 120 python scripts/time_gemm.py ${SHAPES:-16 22016 4096 16 4096 11008 16 4096 4096}; done 2>&1 | tee gpurun_out/cmp.txt
true
