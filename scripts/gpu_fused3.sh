cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
timeout 600 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -2
FIREQ_FFN_PERSISTENT=1 timeout 600 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-prefill > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('FFN', d['value'], 'fused', d['fused_ffn_api_us'])"
