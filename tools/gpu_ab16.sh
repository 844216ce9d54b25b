python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for wv in 0 1 2 3; do
  for wl in 1024 4096; do
    echo "== waves $wv wl $wl" >> gpurun_out/sweep16.log
    PSCWIN_SCAN_WAVES=$wv timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass|"scan_carry|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep16.log
  done
done
cat gpurun_out/sweep16.log
