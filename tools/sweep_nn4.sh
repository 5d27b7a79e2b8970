cd /root/repo
echo "baseline"; python tools/time_roots.py 2>&1 | tail -1
for st in 2 3; do
  echo "wm4 nw4 stages $st occ"; CPKIT_PLAN_DEBUG=1 CPKIT_GRID_OCC=1 CPKIT_NN_WM=4 CPKIT_NN_NW=4 CPKIT_NN_STAGES=$st python tools/time_roots.py 2>&1 | grep -E "plan NN M=160000|back" | sort | uniq | tail -2
done
echo "wm8 nw8 stages 2 occ (2 CTA?)"; CPKIT_GRID_OCC=1 CPKIT_NN_STAGES=2 python tools/time_roots.py 2>&1 | tail -1
echo "C4 baseline"; python tools/time_roots.py 100,100,100,100 50 2>&1 | tail -1
echo "C5s baseline"; python tools/time_roots.py 200,200,200,200 200 2>&1 | tail -1
