python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --breakdown --no-cpu-baseline > gpurun_out/bench1024.log 2>&1
timeout 300 python bench.py --workload 4096 --steps 20 --breakdown --no-cpu-baseline > gpurun_out/bench4096.log 2>&1
timeout 300 python bench.py --workload 4096 --steps 20 --breakdown --no-cpu-baseline --ffn > gpurun_out/bench4096_ffn.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; for f in gpurun_out/bench1024.log gpurun_out/bench4096.log gpurun_out/bench4096_ffn.log; do grep -E '"gemm_out|gemm_fc2|"metric"' $f | cut -c1-180; done
