python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline --breakdown > gpurun_out/ab9_1024_$i.log 2>&1; done
timeout 300 python bench.py --workload 4096 --steps 20 --no-cpu-baseline --breakdown > gpurun_out/ab9_4096.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'scan_pass[12]|conv_silu|scan_carry|layer_norm' -c 6 -o gpurun_out/scan4096_r01h -f python tools/run_stage.py 1 4096 > gpurun_out/scan4096.log 2>&1
tail -n 2 gpurun_out/ab_tests.log; tail -n 1 gpurun_out/smoke.log
