#!/bin/bash
# One parameterised A/B sweep (replaces the round-1 one-off gpu_ab*.sh scripts). Run under gpurun:
#
#   tools/gpu_sweep.sh <name> <kind> "<v1>" "<v2>" ... [-- <workloads>]
#
#   kind = env:<VAR>     each value sets the runtime knob VAR (read once per process by the library)
#   kind = flag:<MACRO>  each value rebuilds the library with -D<MACRO>=<value>
#
# For every value and workload (default: 1024 4096) it runs bench.py --breakdown and appends the step time and
# the per-kernel ms/launch to gpurun_out/<name>.log. A "flag:" sweep also runs the GPU tests of the touched area
# (PSCWIN_SWEEP_TESTS, default tests/test_gpu_scan.py) at each value and appends their summary line.
set -u
name=$1; kind=$2; shift 2
vals=(); wls="1024 4096"
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; wls="$*"; break; fi
  vals+=("$1"); shift
done
log=gpurun_out/$name.log
mkdir -p gpurun_out
for v in "${vals[@]}"; do
  envs=""
  case $kind in
    env:*)  envs="${kind#env:}=$v" ;;
    flag:*) PSCWIN_NVCC_FLAGS="-D${kind#flag:}=$v" python paper_2407_02109_b200/_build.py --force > /dev/null 2>&1 \
              || { echo "== $kind=$v: build failed" >> "$log"; continue; }
            timeout 900 python -m pytest ${PSCWIN_SWEEP_TESTS:-tests/test_gpu_scan.py} -x -q -m gpu > gpurun_out/$name.tests.log 2>&1
            echo "== $kind=$v tests: $(tail -n 1 gpurun_out/$name.tests.log)" >> "$log" ;;
  esac
  for wl in $wls; do
    echo "== $kind=$v workload $wl" >> "$log"
    env $envs timeout 600 python bench.py --workload "$wl" --steps 30 --warmup 5 --no-cpu-baseline --breakdown 2>&1 \
      | python -c "
import json, sys
for l in sys.stdin:
    try:
        d = json.loads(l)
    except Exception:
        continue
    if 'kernel' in d:
        print('   %-22s %9.4f ms/launch  frac %s' % (d['kernel'], d['ms_per_launch'], d.get('frac')))
    elif 'metric' in d:
        print('   STEP %s ms/image' % d['value'])" >> "$log"
  done
done
case $kind in flag:*) python paper_2407_02109_b200/_build.py --force > /dev/null 2>&1 ;; esac
cat "$log"
