python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "qkv or layer_forward" > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2 3; do
  for E in "" "PSCWIN_QKV_PAIR_SMALL=1"; do
    echo "== [$E]" >> gpurun_out/sweep25.log
    env $E timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline --breakdown 2>&1 | grep -E '"gemm_qkv|"metric"' | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print('  ', d.get('kernel','STEP'), d.get('ms_per_launch', d.get('value')))" >> gpurun_out/sweep25.log
  done
done
tail -n 2 gpurun_out/ab_tests.log; cat gpurun_out/sweep25.log
