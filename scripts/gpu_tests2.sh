cd $GRAFT_REPO_ROOT
make -C paper_2505_20839_b200/csrc -j8 all > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --colpar --steps 400 --warmup 8 > gpurun_out/colpar.json 2> gpurun_out/colpar.err; echo "colpar rc=$?"; cat gpurun_out/colpar.json; tail -3 gpurun_out/colpar.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 400 --warmup 8 --no-cpu --no-prefill > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo "torchrun rc=$?"; tail -c 300 gpurun_out/torchrun1.json
