#!/bin/bash
# Tile-shape sweep for the root GEMMs (C2 unless args given).
D=${1:-400,400,400}; R=${2:-100}
for cfg in "WM=5 WN=2 NTW=7" "WM=5 WN=1 NTW=13" "WM=8 WN=1 NTW=13" "WM=7 WN=1 NTW=13" "WM=4 WN=2 NTW=7" "WM=5 WN=2 NTW=7 STAGES=3" "WM=5 WN=2 NTW=7 STAGES=5"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CPKIT_TN_\1=/g') python tools/time_roots.py $D $R | sed "s/^/TN[$cfg] /"
done
for cfg in "WM=8 WN=1 NTW=13" "WM=6 WN=1 NTW=13" "WM=8 WN=1 NTW=13 STAGES=2" "WM=8 WN=1 NTW=13 STAGES=4" "WM=4 WN=2 NTW=7"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CPKIT_NN_\1=/g') python tools/time_roots.py $D $R | sed "s/^/NN[$cfg] /"
done
