# Round profile bundle (outputs under gpurun_out/, summarised into profiles/ by tools/ncu_summary.py):
#   launch list of eager bench steps (cold-cache, serialised per-launch times) and one --set full capture of an
#   eager 1024^2 step (per-kernel DRAM bytes -> profiles/dram_traffic.json for bench.py roofline.traffic)
TAG=${1:-r01h}
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-graph --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -o gpurun_out/full_$TAG -f \
    python tools/run_stage.py 1 1024 > gpurun_out/full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'scan_pass2|window_attn_ws' -c 2 \
    -o gpurun_out/full4096_$TAG -f python tools/run_stage.py 1 4096 > gpurun_out/full4096_$TAG.log 2>&1
python bench.py > gpurun_out/bench1024_$TAG.log 2>&1
python bench.py --workload 4096 --steps 20 --no-cpu-baseline > gpurun_out/bench4096_$TAG.log 2>&1
python bench.py --workload 2048 --steps 10 --no-cpu-baseline > gpurun_out/bench2048_$TAG.log 2>&1
python bench.py --workload ms --steps 10 --no-cpu-baseline > gpurun_out/bench_ms_$TAG.log 2>&1
python bench.py --encoder --steps 20 --no-cpu-baseline > gpurun_out/encoder1024_$TAG.log 2>&1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/reference_$TAG.log 2>&1
ls gpurun_out
