python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PSCWIN_XPROJ_SPLITS=4 timeout 600 python -m pytest tests/test_gpu_scan.py -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do
  for sp in 1 2 3 4; do
    echo "== splits $sp" >> gpurun_out/sweep26.log
    PSCWIN_XPROJ_SPLITS=$sp timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline --breakdown 2>&1 | grep -E '"gemm_x_proj|"xproj_split|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep26.log
  done
done
tail -n 2 gpurun_out/ab_tests.log; cat gpurun_out/sweep26.log
