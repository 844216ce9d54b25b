for c in 1 2; do echo "== case $c"; NCCL_DEBUG=WARN timeout 150 python tools/debug_nccl.py $c 2>&1 | tail -30; done > gpurun_out/debug_nccl.log 2>&1
cat gpurun_out/debug_nccl.log
