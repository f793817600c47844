timeout 200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 100 python tools/knob_sweep.py --format csr_lb --knobs "lb_tile=16384" > gpurun_out/knobs12.txt 2>&1
timeout 100 python tools/knob_sweep.py --matrix powerlaw --format csr_lb,hybrid,csr_classical > gpurun_out/knobs12.txt 2>&1
