timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/knob_sweep.py --matrix 7pt --grid 256 --format csr_classical --knobs "classical_per_sm=16,32" > gpurun_out/knobs17.txt 2>&1
timeout 300 python bench.py --workload c5 --grid 256 --no-cpu > gpurun_out/b_c5g256.log 2>&1
