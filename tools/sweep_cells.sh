#!/bin/bash
# Root-GEMM tile sweep: planner default, then each override set given as
#   KIND:WM,NW,NT8[,STAGES]   (KIND = NN or TN; env CPKIT_<KIND>_*)
# Usage: tools/sweep_cells.sh DIMS RANK CFG...   e.g. 400,400,400 100 NN:8,8,13 TN:5,8,13
cd "$(dirname "$0")/.."
D=${1:-400,400,400}; R=${2:-100}; shift 2 2>/dev/null
echo "default: $(python tools/time_roots.py $D $R 2>&1 | tail -1)"
for cfg in "$@"; do
  kind=${cfg%%:*}; IFS=, read -r wm nw nt st <<< "${cfg#*:}"
  env CPKIT_${kind}_WM=$wm CPKIT_${kind}_NW=$nw CPKIT_${kind}_NT8=$nt ${st:+CPKIT_${kind}_STAGES=$st} \
    timeout 120 python tools/time_roots.py $D $R 2>&1 | tail -1 | sed "s/^/$cfg /"
done
