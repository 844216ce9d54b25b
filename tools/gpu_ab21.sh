python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_attn.py > gpurun_out/dbg21.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg21.log
if grep -q "ok 1" gpurun_out/dbg21.log; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_ms.py tests/test_gpu_ends.py -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
  for wl in 1024 2048 4096; do timeout 300 python bench.py --workload $wl --steps 20 --no-cpu-baseline --breakdown > gpurun_out/ab21_$wl.log 2>&1; done
  timeout 300 python tools/attn_timeline.py 256 > gpurun_out/attn_tl_256_d.log 2>&1
fi
cat gpurun_out/dbg21.log; tail -n 2 gpurun_out/ab_tests.log
