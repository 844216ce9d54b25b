# one gpurun session: benches (outputs under gpurun_out/)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --breakdown --no-cpu-baseline > gpurun_out/bench1024.log 2>&1
PSCWIN_NO_SIDE_STREAM=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench1024_noside.log 2>&1
timeout 600 python bench.py --breakdown --no-cpu-baseline --ffn > gpurun_out/bench1024_ffn.log 2>&1
timeout 600 python bench.py --workload 4096 --steps 20 --breakdown --no-cpu-baseline --ffn > gpurun_out/bench4096_ffn.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 1 $f | cut -c1-300; done
