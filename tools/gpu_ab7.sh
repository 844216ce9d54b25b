python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline > gpurun_out/ab7_pdl_$i.log 2>&1; PSCWIN_PDL=0 timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline > gpurun_out/ab7_nopdl_$i.log 2>&1; done
timeout 300 python bench.py --workload 2048 --steps 10 --no-cpu-baseline > gpurun_out/ab7_2048.log 2>&1
PSCWIN_PDL=0 timeout 300 python bench.py --workload 2048 --steps 10 --no-cpu-baseline > gpurun_out/ab7_2048_nopdl.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'gemm_bf16_kernelILb.ELi3E' -c 2 -o gpurun_out/xproj1024 -f python tools/run_stage.py 1 1024 > gpurun_out/ncu_x.log 2>&1
tail -n 2 gpurun_out/ab_tests.log; cat gpurun_out/smoke.log | tail -n 1
