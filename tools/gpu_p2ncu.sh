python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
$N -k regex:'scan_pass2' -c 1 -o gpurun_out/pass2_1024_final -f python tools/run_stage.py 1 1024 > /dev/null 2>&1
$N -k regex:'scan_pass2' -c 1 -o gpurun_out/pass2_4096_final -f python tools/run_stage.py 1 4096 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-graph --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/*final*
