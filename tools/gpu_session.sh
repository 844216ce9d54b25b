python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ends.py -q > gpurun_out/pytest_ends.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f | cut -c1-300; done
