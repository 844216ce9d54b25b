python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ls in auto 0 1; do
  for wl in 1024 2048 4096; do
    echo "== lockstep $ls wl $wl" >> gpurun_out/sweep20.log
    E=""; [ "$ls" != auto ] && E="PSCWIN_ATTN_LOCKSTEP=$ls"
    env $E timeout 300 python bench.py --workload $wl --steps 20 --no-cpu-baseline --breakdown 2>&1 | grep -E '"window_attention|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep20.log
  done
done
cat gpurun_out/sweep20.log
