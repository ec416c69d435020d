# quick iteration: GPU parity tests + decode GEMM timings (+ optional trace)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 120 python scripts/time_gemm.py 16 22016 4096 16 4096 11008 16 4096 4096 16 14336 4096 16 4096 14336 2>&1 | tee gpurun_out/time.txt
[ -n "$TRACE" ] && FIREQ_DEBUG_MODE=64 timeout 100 python scripts/trace_gemm.py 16 22016 4096 2>&1 | head -24
true
