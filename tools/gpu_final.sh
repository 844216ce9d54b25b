python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo rc=$? >> gpurun_out/final_tests.log
python bench.py > gpurun_out/final_bench1024.log 2>&1
python bench.py --workload 4096 --steps 20 --no-cpu-baseline > gpurun_out/final_bench4096.log 2>&1
python bench.py --workload 2048 --steps 10 --no-cpu-baseline > gpurun_out/final_bench2048.log 2>&1
python bench.py --shard rows --workload 4096 --steps 10 --no-cpu-baseline > gpurun_out/final_rows4096.log 2>&1
tail -n 2 gpurun_out/final_tests.log; tail -n 1 gpurun_out/smoke.log
