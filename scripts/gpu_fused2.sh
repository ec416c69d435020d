cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
timeout 600 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 > gpurun_out/pytest_ffn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ffn.log
tail -5 gpurun_out/pytest_ffn.log
timeout 300 python bench.py --no-cpu --no-prefill > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('FFN', d['value'], 'fused', d['fused_ffn_api_us'])"
FIREQ_FFN_2KERNELS=1 timeout 300 python bench.py --no-cpu --no-prefill > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python -c "import json; d=json.load(open('gpurun_out/bench2.json')); print('2-kernel fused', d['fused_ffn_api_us'])"
for w in 1 2; do FIREQ_TRACE_WHICH=$w timeout 120 python scripts/chain_trace_fused.py 2>&1 | tail -20 | head -16; done
