python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for wl in 1024 4096; do timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab3_bench$wl.log 2>&1; done
tail -n 3 gpurun_out/ab_tests.log
