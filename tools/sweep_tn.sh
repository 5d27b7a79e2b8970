cd /root/repo
python tools/time_roots.py
for cfg in "5 1 13" "5 2 7" "8 1 13" "4 1 13" "4 2 7" "10 1 13" "5 1 13 3" "8 1 13 3"; do
  set -- $cfg
  if [ -n "$4" ]; then export CPKIT_TN_STAGES=$4; else unset CPKIT_TN_STAGES; fi
  echo "wm=$1 wn=$2 ntw=$3 stages=${4:-auto}: $(CPKIT_TN_WM=$1 CPKIT_TN_WN=$2 CPKIT_TN_NTW=$3 timeout 120 python tools/time_roots.py 2>&1 | tail -1)"
done
