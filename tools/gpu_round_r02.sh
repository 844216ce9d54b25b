#!/bin/bash
# Round-2 measurement bundle (outputs under gpurun_out/, which must stay < 64 MiB to come back; summaries go to
# profiles/r02/ via tools/ncu_summary.py): the default bench line (4096^2 north-star stack) and the 1024^2 / 2048^2
# lines, the partition / merge GB/s micro-benchmark, the ncu launch list of the default bench command, and one
# --set full capture of the kernels matching $KREGEX over the first three layers of an eager 4096^2 step (raw CSV
# exported on the box; the .ncu-rep is kept only when small).
TAG=${1:-r02}
KREGEX=${2:-gemm_bf16}
KCOUNT=${3:-10}
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 20 --warmup 5 --breakdown > gpurun_out/bench4096_$TAG.log 2>&1
python bench.py --workload 1024 --steps 30 --no-cpu-baseline --breakdown > gpurun_out/bench1024_$TAG.log 2>&1
python bench.py --workload 2048 --steps 10 --no-cpu-baseline > gpurun_out/bench2048_$TAG.log 2>&1
python bench.py --micro partition --steps 20 > gpurun_out/micro_partition_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4096_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches4096_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -c $KCOUNT -o /tmp/full4096_$TAG -f \
    python tools/run_stage.py 1 4096 > gpurun_out/full4096_$TAG.log 2>&1
ncu -i /tmp/full4096_$TAG.ncu-rep --page raw --csv > gpurun_out/full4096_${TAG}_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/full4096_$TAG.ncu-rep gpurun_out/traffic4096_$TAG.json > gpurun_out/full4096_${TAG}_summary.md 2>&1
sz=$(stat -c %s /tmp/full4096_$TAG.ncu-rep 2>/dev/null || echo 0)
[ "$sz" -lt 30000000 ] && cp /tmp/full4096_$TAG.ncu-rep gpurun_out/
du -sh gpurun_out
