run() {
  for wl in 1024 4096; do
    timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass2|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  $wl', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep19.log
  done
}
python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
echo "== NS2=2 default" >> gpurun_out/sweep19.log; run
echo "== NS2=4 MINB4=1" >> gpurun_out/sweep19.log; PSCWIN_SCAN_NS2=4 run
for m in 3 4; do
  PSCWIN_NVCC_FLAGS="-DPSCWIN_PASS2_MINB4=$m" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  echo "== NS2=4 MINB4=$m" >> gpurun_out/sweep19.log; PSCWIN_SCAN_NS2=4 run
done
cat gpurun_out/sweep19.log
