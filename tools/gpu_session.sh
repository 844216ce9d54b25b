set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --breakdown > gpurun_out/bench1024.log 2>&1
timeout 600 python bench.py --workload 2048 --steps 20 --no-cpu-baseline --breakdown > gpurun_out/bench2048.log 2>&1
timeout 600 python bench.py --workload 4096 --steps 20 --no-cpu-baseline --breakdown > gpurun_out/bench4096.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/*.log
