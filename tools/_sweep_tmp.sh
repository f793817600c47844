timeout 300 python -m pytest tests/test_solvers_gpu.py -x -q > gpurun_out/t_solv.log 2>&1
for f in 1 0; do
  B200SP_FUSED_SPMV_DOT=$f timeout 300 python bench.py --workload c4b --no-cpu > gpurun_out/b_c4b_f$f.log 2>&1
  B200SP_FUSED_SPMV_DOT=$f timeout 300 python bench.py --workload c5 --no-cpu --grid 256 > gpurun_out/b_c5g256_f$f.log 2>&1
done
