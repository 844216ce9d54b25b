# one gpurun session: parity tests, benches (outputs under gpurun_out/)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --breakdown --no-cpu-baseline > gpurun_out/bench1024.log 2>&1
PSCWIN_DT_FFMA=1 timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench1024_dtffma.log 2>&1
timeout 600 python bench.py --workload 4096 --steps 20 --breakdown --no-cpu-baseline > gpurun_out/bench4096.log 2>&1
timeout 1200 python bench.py --ablation --steps 10 > gpurun_out/ablation.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 1 $f | cut -c1-200; done
