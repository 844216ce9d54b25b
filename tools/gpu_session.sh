# one gpurun session: parity tests, benches, launch list (outputs under gpurun_out/)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ms.py -x -q > gpurun_out/pytest_ms.log 2>&1; echo pytest rc $?
timeout 900 python bench.py --workload ms --steps 10 --breakdown > gpurun_out/bench_ms.log 2>&1
timeout 600 python bench.py --breakdown --no-cpu-baseline > gpurun_out/bench1024.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
