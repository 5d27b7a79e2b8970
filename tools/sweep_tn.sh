cd /root/repo
for shape in "400,400,400 100" "100,100,100,100 50" "200,200,200 20"; do
python tools/time_roots.py $shape
for cfg in "4 2 7" "5 2 7" "6 2 7" "8 1 13" "4 1 7" "8 1 7"; do
  set -- $cfg
  echo "wm=$1 wn=$2 ntw=$3: $(CPKIT_TN_WM=$1 CPKIT_TN_WN=$2 CPKIT_TN_NTW=$3 timeout 120 python tools/time_roots.py $shape 2>&1 | tail -1)"
done
done
