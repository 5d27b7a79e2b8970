cd /root/repo
python tools/time_roots.py 100,100,100,100 50
for cfg in "8 1 7" "6 1 7" "4 1 7" "8 2 4" "4 2 4" "10 1 7" "8 1 8" "6 2 4"; do
  set -- $cfg
  echo "NN wm=$1 wn=$2 ntw=$3: $(CPKIT_NN_WM=$1 CPKIT_NN_WN=$2 CPKIT_NN_NTW=$3 timeout 120 python tools/time_roots.py 100,100,100,100 50 2>&1 | tail -1 | sed 's/dims=.*env=[^ ]* //')"
done
for cfg in "8 1 8" "8 2 4" "4 2 4" "10 1 7"; do
  set -- $cfg
  echo "TN wm=$1 wn=$2 ntw=$3: $(CPKIT_TN_WM=$1 CPKIT_TN_WN=$2 CPKIT_TN_NTW=$3 timeout 120 python tools/time_roots.py 100,100,100,100 50 2>&1 | tail -1 | sed 's/dims=.*env=[^ ]* //')"
done
