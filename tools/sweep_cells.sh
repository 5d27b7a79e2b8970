# Root GEMM tile sweep (cell-run kernel): planner default vs overrides
cd /root/repo
python tools/time_roots.py 2>&1 | tail -1
for cfg in "NN 8 8 13" "NN 4 8 13" "NN 4 8 14" "NN 6 12 13" "NN 8 12 13" "TN 5 8 13" "TN 4 8 14" "TN 5 12 13"; do
  set -- $cfg
  echo "$1 wm=$2 nw=$3 nt8=$4: $(env CPKIT_$1_WM=$2 CPKIT_$1_NW=$3 CPKIT_$1_NT8=$4 timeout 120 python tools/time_roots.py 2>&1 | tail -1)"
done
