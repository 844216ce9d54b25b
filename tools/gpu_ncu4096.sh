# one --set full capture per kernel of interest at 4096^2 (run_stage.py: one eager 12-layer step)
python -c "import __graft_entry__ as g; g.build()"
N="ncu --set full --clock-control none --import-source on"
$N -k regex:'gemm_bf16_kernelILb.ELi3E' -s 1 -c 1 -o gpurun_out/dt4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_dt.log 2>&1
$N -k regex:conv_silu -c 1 -o gpurun_out/conv4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_conv.log 2>&1
$N -k regex:window_attn_ws -s 1 -c 1 -o gpurun_out/attn4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_attn.log 2>&1
$N -k regex:'gemm_bf16_kernelILb.ELi0E' -s 2 -c 1 -o gpurun_out/oproj4096 -f python tools/run_stage.py 1 4096 > gpurun_out/ncu_oproj.log 2>&1
ls -la gpurun_out/*.ncu-rep
