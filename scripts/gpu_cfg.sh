# FFN bench + gate_up / down trace per FIREQ_CFG16 variant
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
for v in ${VARIANTS:-0 1 2 3 4}; do
  echo "=== FIREQ_CFG16=$v"
  FIREQ_CFG16=$v timeout 200 python bench.py --no-cpu --no-prefill --steps 1000 > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_v$v.json')); print('FFN', d['value'], 'gu', d['roofline']['launch_us'], 'down', d['gemm_down']['us'])"
  FIREQ_CFG16=$v timeout 300 python scripts/trace_gemm.py 2>&1 | grep -E "^M=16 N=(22016|4096) K=(4096|11008)" -A 8 | grep -E "^M=|first_data|mma_done|end "
done
