timeout 200 python tools/knob_sweep.py --format csr_lb --knobs "lb2_unroll=4,1 lb_tile=16384,32768,65536" > gpurun_out/knobs19.txt 2>&1
timeout 200 python tools/knob_sweep.py --dtype float32 --format csr_lb --knobs "lb2_unroll=4,1 lb_tile=16384,65536" >> gpurun_out/knobs19.txt 2>&1
timeout 300 python tools/knob_sweep.py --matrix 7pt --grid 256 --format csr_lb --knobs "lb2_unroll=4,1 lb_tile=16384,65536" >> gpurun_out/knobs19.txt 2>&1
