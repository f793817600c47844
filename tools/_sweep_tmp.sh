timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bench_torchrun.log 2>&1
