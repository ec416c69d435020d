# A/B: current libfireq.so vs libfireq_prev.so (the previous commit), same process order alternated
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for lib in libfireq_prev.so libfireq.so; do echo "== $lib"; LIB=paper_2505_20839_b200/$lib timeout 120 python scripts/time_gemm.py ${SHAPES:-16 22016 4096 16 4096 11008 16 4096 4096 16 14336 4096}; done
done 2>&1 | sed 's/plan=.*e}//' | tee gpurun_out/ab.txt
