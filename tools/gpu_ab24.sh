python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  for E in "" "PSCWIN_PDL_EVEN=1"; do
    for wl in 1024 4096; do
      echo "== [$E] $wl" >> gpurun_out/sweep24.log
      env $E timeout 300 python bench.py --workload $wl --steps 50 --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  ', d['value'])" >> gpurun_out/sweep24.log
    done
  done
done
cat gpurun_out/sweep24.log
