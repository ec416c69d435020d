# tests + A/B bench of an env toggle (AB_ENV, e.g. FIREQ_NO_CSPLIT=1)
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/trace_gemm.py 2>&1 | tail -12
for i in 1 2; do
  timeout 600 python bench.py --no-cpu --no-prefill > gpurun_out/bench_a$i.json 2> gpurun_out/bench_a$i.err
  cat gpurun_out/bench_a$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['value'], d['roofline'])"
  env ${AB_ENV} timeout 600 python bench.py --no-cpu --no-prefill > gpurun_out/bench_b$i.json 2> gpurun_out/bench_b$i.err
  cat gpurun_out/bench_b$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['value'], d['roofline'])"
done
