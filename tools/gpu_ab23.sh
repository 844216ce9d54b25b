python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ends.py tests/test_gpu_f32.py -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline --breakdown > gpurun_out/ab23_1024_$i.log 2>&1; done
timeout 300 python bench.py --workload 4096 --steps 20 --no-cpu-baseline --breakdown > gpurun_out/ab23_4096.log 2>&1
tail -n 2 gpurun_out/ab_tests.log
