# profiling session: launch list of the bench step + one ncu --set full capture (outputs under gpurun_out/)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -o gpurun_out/step_full -f \
  python tools/run_stage.py 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.md 2>&1
python tools/ncu_summary.py full gpurun_out/step_full.ncu-rep gpurun_out/dram_traffic.json > gpurun_out/full_step.md 2>&1
tail -3 gpurun_out/ncu_full.log; cat gpurun_out/launches.md gpurun_out/full_step.md
