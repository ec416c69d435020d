# FFN bench for combinations: ENVSETS="A=1,B=2 A=3" (comma-separated env assignments per run)
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all > /dev/null
for set in ${ENVSETS}; do
  envs=$(echo $set | tr ',' ' ')
  env $envs timeout 200 python bench.py --no-cpu --no-prefill --steps 2000 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_e.json')); print('$set', 'FFN', d['value'], 'fused', d.get('fused_ffn_api_us'), 'gu', d['roofline']['launch_us'], 'down', d['gemm_down']['us'])" || tail -2 gpurun_out/bench_e.err
done
