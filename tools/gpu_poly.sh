# polynomial-exp2 offload sweep for the scan passes + attention timeline at 4096^2 (outputs under gpurun_out/)
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py -x -q > gpurun_out/poly_tests.log 2>&1; echo rc=$? >> gpurun_out/poly_tests.log
for cfg in "0 0" "4 8" "2 8" "4 4" "2 4"; do
  set -- $cfg
  echo "== poly1 $1 poly2 $2" >> gpurun_out/poly.log
  PSCWIN_SCAN_POLY1=$1 PSCWIN_SCAN_POLY2=$2 timeout 300 python bench.py --workload 4096 --steps 20 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  if 'kernel' in d: print('  %-12s %.4f ms/launch frac %.3f'%(d['kernel'],d['ms_per_launch'],d.get('frac',0)))
  else: print('  value', d['value'])" >> gpurun_out/poly.log
done
timeout 300 python tools/attn_timeline.py 256 > gpurun_out/attn_tl_256.log 2>&1
cat gpurun_out/poly_tests.log | tail -3; cat gpurun_out/poly.log
