# per-CTA traces, CTA-0 event log and the FFN span timeline (profile build)
cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all prof > /dev/null
timeout 300 python scripts/trace_gemm.py > gpurun_out/trace.txt 2>&1
timeout 300 python scripts/evt_gemm.py 16 22016 4096 > gpurun_out/evt_gu.txt 2>&1
timeout 300 python scripts/evt_gemm.py 16 4096 11008 > gpurun_out/evt_down.txt 2>&1
timeout 300 python scripts/span_ffn.py > gpurun_out/span.txt 2>&1
