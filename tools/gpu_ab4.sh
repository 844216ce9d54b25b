python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --workload 4096 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab4_base.log 2>&1
PSCWIN_GEMM_PAIR=0 timeout 300 python bench.py --workload 4096 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab4_nopair.log 2>&1
PSCWIN_GEMM_PAIR=0 timeout 300 python bench.py --workload 1024 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab4_nopair1024.log 2>&1
timeout 300 python bench.py --workload 1024 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab4_base1024.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'scan_pass2' -c 1 -o gpurun_out/pass2_4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_p2.log 2>&1
$N -k regex:'gemm_bf16_kernelILb.ELi3E' -s 1 -c 1 -o gpurun_out/dt4096b -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_dt.log 2>&1
