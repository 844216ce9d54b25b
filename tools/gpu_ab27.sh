for t in 16 8 32; do
  PSCWIN_NVCC_FLAGS="-DPSCWIN_TSUB=$t" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  if [ $t = 8 ]; then PSCWIN_NVCC_FLAGS="-DPSCWIN_TSUB=8" timeout 600 python -m pytest tests/test_gpu_scan.py -x -q -k "not 4096" > gpurun_out/tsub_tests.log 2>&1; tail -n 1 gpurun_out/tsub_tests.log >> gpurun_out/sweep27.log; fi
  for wl in 1024 4096; do
    echo "== TSUB $t wl $wl" >> gpurun_out/sweep27.log
    timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"scan_pass|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep27.log
  done
done
cat gpurun_out/sweep27.log
