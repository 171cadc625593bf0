#!/bin/bash
# A/B timing of the headline bench under environment switches:
#   tools/ab.sh TAG [BENCH_ARGS --] "ENV=.. ENV2=.." ...
# one line per variant into gpurun_out/TAG.txt (ms per step)
out=gpurun_out/$1.txt; shift
extra=""
if [[ "$*" == *" -- "* ]] || [[ "$1" == --* ]]; then
  while [[ "$1" != "--" ]]; do extra="$extra $1"; shift; done; shift
fi
: > $out
for cfg in "$@"; do
  r=$(env $cfg timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-strong --no-baselines --no-cpu-baseline --soak-ms 300 $extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>&1)
  echo "$cfg $r" >> $out
done
