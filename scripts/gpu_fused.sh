# fused FFN: tests + bench + chain spans
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
timeout 600 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 > gpurun_out/pytest_ffn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ffn.log
tail -15 gpurun_out/pytest_ffn.log
timeout 600 python bench.py --no-cpu --no-prefill > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
