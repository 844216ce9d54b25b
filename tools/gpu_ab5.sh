python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for wl in 1024 4096; do timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab5_bench$wl.log 2>&1; done
PSCWIN_NO_SIDE_STREAM=1 timeout 300 python bench.py --workload 4096 --steps 30 --no-cpu-baseline > gpurun_out/ab5_noside4096.log 2>&1
PSCWIN_NO_SIDE_STREAM=1 timeout 300 python bench.py --workload 1024 --steps 30 --no-cpu-baseline > gpurun_out/ab5_noside1024.log 2>&1
timeout 300 python tools/attn_timeline.py 256 > gpurun_out/attn_tl_256_c.log 2>&1
tail -n 3 gpurun_out/ab_tests.log
