python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do timeout 300 python bench.py --workload 1024 --steps 100 --no-cpu-baseline --breakdown > gpurun_out/ab10_1024_$i.log 2>&1; done
timeout 300 python bench.py --workload 4096 --steps 20 --no-cpu-baseline --breakdown > gpurun_out/ab10_4096.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'scan_pass2' -c 1 -o gpurun_out/pass2_4096_r01h -f python tools/run_stage.py 1 4096 > gpurun_out/p2_4096.log 2>&1
PSCWIN_XPROJ_SPLITS=4 $N -k regex:'gemm_bf16_kernelILb.ELi3E' -c 1 -o gpurun_out/xproj_split4 -f python tools/run_stage.py 1 1024 > gpurun_out/xs.log 2>&1
tail -n 2 gpurun_out/ab_tests.log
