for m in 3 0 2 4; do
  PSCWIN_NVCC_FLAGS="-DPSCWIN_ATTN_POLY_MOD=$m" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  for wl in 1024 4096; do
    echo "== poly_mod $m wl $wl" >> gpurun_out/sweep22.log
    timeout 300 python bench.py --workload $wl --steps 20 --no-cpu-baseline --breakdown 2>&1 | grep -E '"window_attention|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep22.log
  done
done
cat gpurun_out/sweep22.log
