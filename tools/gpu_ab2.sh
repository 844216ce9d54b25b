# A/B: attention TMA-store + pipelined softmax loads, scan staging without delta_low, pass-2 MINB 5 vs 6
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
timeout 300 python tools/attn_timeline.py 256 > gpurun_out/attn_tl_256_b.log 2>&1
for wl in 1024 4096; do timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab_bench$wl.log 2>&1; done
PSCWIN_ATTN_DIRECT_STORE=1 timeout 300 python bench.py --workload 4096 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab_bench4096_direct.log 2>&1
PSCWIN_NVCC_FLAGS="-DPSCWIN_PASS2_MINB=6" python -m paper_2407_02109_b200._build --force > /dev/null 2>&1
for wl in 1024 4096; do timeout 300 python bench.py --workload $wl --steps 30 --no-cpu-baseline --breakdown > gpurun_out/ab_bench${wl}_minb6.log 2>&1; done
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'gemm_bf16_kernelILb.ELi3E' -s 1 -c 1 -o gpurun_out/dt4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_dt.log 2>&1
$N -k regex:'gemm_bf16_kernelILb.ELi0E' -s 2 -c 1 -o gpurun_out/inproj4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_inproj.log 2>&1
tail -n 3 gpurun_out/ab_tests.log
