timeout 300 python -m pytest tests/test_spmv_gpu.py -q -x -k "coo or hybrid" > gpurun_out/t_coo.log 2>&1
timeout 200 python tools/knob_sweep.py --format coo,hybrid --knobs "coo_minb=1,6" > gpurun_out/knobs18.txt 2>&1
timeout 200 python tools/knob_sweep.py --dtype float32 --format coo --knobs "coo_minb=1,6" >> gpurun_out/knobs18.txt 2>&1
timeout 200 python tools/knob_sweep.py --matrix powerlaw --format coo,hybrid >> gpurun_out/knobs18.txt 2>&1
