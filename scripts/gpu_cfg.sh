# steady-state slope vs fixed overhead of the decode GEMM: N sweep, L2-resident (ROT=1) vs HBM (ROT=4)
cd $GRAFT_REPO_ROOT
for v in ${CFGS:-0 1}; do for r in 1 4; do echo "== cfg $v ROT=$r"; FIREQ_CFG16=$v ROT=$r timeout 120 python scripts/time_gemm.py 16 5504 4096 16 11008 4096 16 22016 4096 16 44032 4096 16 88064 4096; done; done 2>&1 | tee gpurun_out/cfg.txt
