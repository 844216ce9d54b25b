# pass-2 unroll / occupancy sweep (rebuilds with PSCWIN_NVCC_FLAGS)
for cfg in "-DPSCWIN_PASS2_MINB=4 -DPSCWIN_P2_UNROLL=8" "-DPSCWIN_PASS2_MINB=4 -DPSCWIN_P2_UNROLL=16" "-DPSCWIN_PASS2_MINB=3" "-DPSCWIN_PASS2_MINB=3 -DPSCWIN_P2_UNROLL=16" "-DPSCWIN_PASS2_MINB=4"; do
  PSCWIN_NVCC_FLAGS="$cfg" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/sweep14.log
  for wl in 1024 4096; do
    timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass2"|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  $wl', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep14.log
  done
done
cat gpurun_out/sweep14.log
