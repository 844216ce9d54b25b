python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --workload 1024 --steps 50 --no-cpu-baseline --breakdown > gpurun_out/ab6_base.log 2>&1
for s in 2 4; do PSCWIN_XPROJ_SPLITS=$s timeout 300 python bench.py --workload 1024 --steps 50 --no-cpu-baseline --breakdown > gpurun_out/ab6_split$s.log 2>&1; done
PSCWIN_PDL=1 timeout 300 python bench.py --workload 1024 --steps 50 --no-cpu-baseline --breakdown > gpurun_out/ab6_pdl.log 2>&1
PSCWIN_PDL=1 timeout 300 python bench.py --workload 4096 --steps 20 --no-cpu-baseline > gpurun_out/ab6_pdl4096.log 2>&1
