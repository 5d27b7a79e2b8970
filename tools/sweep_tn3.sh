cd /root/repo
python tools/time_roots.py
for cfg in "4 2 7 0" "5 1 13 0" "5 1 13 3" "5 1 13 4" "5 2 7 0" "5 2 7 3" "10 1 13 2" "3 2 7 0"; do
  set -- $cfg
  if [ $4 = 0 ]; then unset CPKIT_TN_STAGES; else export CPKIT_TN_STAGES=$4; fi
  echo "wm=$1 wn=$2 ntw=$3 st=$4: $(CPKIT_TN_WM=$1 CPKIT_TN_WN=$2 CPKIT_TN_NTW=$3 timeout 120 python tools/time_roots.py 2>&1 | tail -1)"
done
