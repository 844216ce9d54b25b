python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "base" "bn128" "bn256" "waves3"; do
  case $cfg in base) E="";; bn128) E="PSCWIN_GEMM_BN=128";; bn256) E="PSCWIN_GEMM_BN=256";; waves3) E="PSCWIN_SCAN_WAVES=3";; esac
  for wl in 1024 4096; do
    echo "== $cfg $wl" >> gpurun_out/sweep17.log
    env $E timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"gemm|"scan_pass|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep17.log
  done
done
cat gpurun_out/sweep17.log
