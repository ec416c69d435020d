# A/B of decode GEMM template configurations (FIREQ_CFG16) and debug modes
cd $GRAFT_REPO_ROOT
for v in ${CFGS:-0}; do for m in ${MODES:-0}; do echo "== cfg $v dbg $m"; FIREQ_CFG16=$v FIREQ_DEBUG_MODE=$m timeout 120 python scripts/time_gemm.py ${SHAPES:-16 5504 4096 16 11008 4096 16 22016 4096 16 44032 4096 16 88064 4096}; done; done 2>&1 | tee gpurun_out/cfg.txt
for v in ${TESTCFGS:-}; do echo "== tests cfg $v"; FIREQ_CFG16=$v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1; done
true
