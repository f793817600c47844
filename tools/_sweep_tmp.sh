timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for w in c1 c3 c4b c4g c5; do timeout 600 python bench.py --workload $w --no-cpu > gpurun_out/bench_$w.log 2>&1; done
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
