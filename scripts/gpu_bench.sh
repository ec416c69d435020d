cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 > /dev/null
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-prefill --no-cpu > /dev/null 2> gpurun_out/ncu_launch.err; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 2 -c 1 -o gpurun_out/prof_gu_m16 python scripts/prof_gemm.py 16 22016 4096 4 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_w4a8_gemm -s 1 -c 1 -o gpurun_out/prof_gu_m16k python scripts/prof_gemm.py 16384 22016 4096 2 > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
