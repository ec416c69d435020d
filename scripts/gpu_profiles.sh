# Round profiles: GPU tests, bench line, ncu launch list of the bench, ncu --set full of the
# decode/prefill GEMMs, C1/C3/C5 sweep.  Outputs under gpurun_out/ (summarised into profiles/).
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python scripts/sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-prefill --no-cpu > /dev/null 2> gpurun_out/ncu_launch.err; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 2 -c 1 -o gpurun_out/prof_gu_m16 python scripts/prof_gemm.py 16 22016 4096 4 > gpurun_out/ncu1.log 2>&1; echo "full1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 2 -c 1 -o gpurun_out/prof_down_m16 python scripts/prof_gemm.py 16 4096 11008 4 > gpurun_out/ncu2.log 2>&1; echo "full2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 1 -c 1 -o gpurun_out/prof_gu_m16k python scripts/prof_gemm.py 16384 22016 4096 2 > gpurun_out/ncu3.log 2>&1; echo "full3 rc=$?"
cat gpurun_out/bench.json
