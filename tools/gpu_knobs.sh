# scan-knob sweep + pipe microbenchmark (outputs under gpurun_out/)
cd tools/ubench && ./pipes > ../../gpurun_out/pipes.log 2>&1; cd ../..
for wl in 1024 4096; do
 for ns2 in 1 2 4; do
  for waves in 1 2; do
   echo "== wl $wl ns2 $ns2 waves $waves" >> gpurun_out/knobs.log
   PSCWIN_SCAN_NS2=$ns2 PSCWIN_SCAN_WAVES=$waves timeout 300 python bench.py --workload $wl --steps 20 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  if 'kernel' in d: print('  %-12s %.4f ms/launch frac %.3f'%(d['kernel'],d['ms_per_launch'],d.get('frac',0)))
  else: print('  value', d['value'])" >> gpurun_out/knobs.log
  done
 done
done
cat gpurun_out/pipes.log gpurun_out/knobs.log
