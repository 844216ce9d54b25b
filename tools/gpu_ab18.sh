for t in 8 4 6 16; do
  PSCWIN_NVCC_FLAGS="-DPSCWIN_CONV_T=$t" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
  for wl in 1024 4096; do
    echo "== CONV_T $t wl $wl" >> gpurun_out/sweep18.log
    timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown 2>&1 | grep -E '"conv_silu|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep18.log
  done
done
PSCWIN_NVCC_FLAGS="-DPSCWIN_CONV_T=4" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_bands.py -x -q > gpurun_out/t4.log 2>&1; tail -n 1 gpurun_out/t4.log >> gpurun_out/sweep18.log
cat gpurun_out/sweep18.log
