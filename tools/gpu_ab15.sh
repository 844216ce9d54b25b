# pass-1 threads-per-channel / occupancy sweep
run() {  # $1 label, env in the caller
  for wl in 1024 4096; do
    timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass1"|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  $wl', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep15.log
  done
}
python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
echo "== NS1=4 default" >> gpurun_out/sweep15.log; run
echo "== NS1=2" >> gpurun_out/sweep15.log; PSCWIN_SCAN_NS1=2 run
for m in 5 6 8; do
  PSCWIN_NVCC_FLAGS="-DPSCWIN_PASS1_MINB=$m" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  echo "== NS1=4 MINB $m" >> gpurun_out/sweep15.log; run
done
cat gpurun_out/sweep15.log
