#!/bin/bash
# One parameterised GPU profiling bundle (replaces the round-1/2 one-off gpu_*.sh scripts). Run under gpurun:
#
#   tools/gpu_profile.sh <tag> [what ...]
#
#   tests     smoke() + the whole GPU test suite                      -> gpurun_out/<tag>_smoke.log, _tests.log
#   bench     bench lines: 4096^2 (default workload), 1024^2, 2048^2   -> gpurun_out/<tag>_bench<wl>.log
#   launches  ncu launch list of the default bench command            -> gpurun_out/<tag>_launches.csv
#   ncu:<re>  one `ncu --set full` capture (mangled-name regex <re>) of an eager 4096^2 step
#                                                                      -> gpurun_out/<tag>_<n>.ncu-rep
#   timeline  attention phase timeline + L2-cold / warm probe         -> gpurun_out/<tag>_attn.log
#   pipes     MUFU / FMA / F2FP / TMEM / exp-pass microbenchmarks     -> gpurun_out/<tag>_ubench.log
#   sanitize  compute-sanitizer memcheck / racecheck / synccheck       -> gpurun_out/<tag>_san_<tool>.log
#
# Knob A/B sweeps: tools/gpu_sweep.sh. Summaries for profiles/: tools/ncu_summary.py, ncu_hot.py, ncu_lines.py.
set -u
tag=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail -20 gpurun_out/${tag}_build.log; exit 1; }
n=0
for w in "$@"; do
  case $w in
    tests)
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
      timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1
      echo "tests: $(tail -n 1 gpurun_out/${tag}_tests.log)" ;;
    bench)
      for wl in 4096 1024 2048; do
        python bench.py --workload $wl --steps 20 --warmup 5 --breakdown > gpurun_out/${tag}_bench$wl.log 2>&1
        echo "bench $wl: $(grep -o '"value": [0-9.]*' gpurun_out/${tag}_bench$wl.log | head -n 1)"
      done ;;
    launches)
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
      python tools/ncu_summary.py launches gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.md 2>&1 ;;
    ncu:*)
      n=$((n + 1))
      ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:${w#ncu:}" -c 1 \
          -o gpurun_out/${tag}_$n -f python tools/run_stage.py 1 4096 > gpurun_out/${tag}_ncu$n.log 2>&1 ;;
    timeline)
      { python tools/attn_timeline.py 256; python tools/attn_l2_probe.py; } > gpurun_out/${tag}_attn.log 2>&1 ;;
    pipes)
      for u in pipes tmem_ld softmax_pass; do
        nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/$u tools/ubench/$u.cu && /tmp/$u
      done > gpurun_out/${tag}_ubench.log 2>&1 ;;
    sanitize)
      for t in memcheck racecheck synccheck; do
        timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py \
            > gpurun_out/${tag}_san_$t.log 2>&1
        echo "$t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${tag}_san_$t.log | tail -n 1)"
      done ;;
    *) echo "unknown item $w" ;;
  esac
done
du -sh gpurun_out
