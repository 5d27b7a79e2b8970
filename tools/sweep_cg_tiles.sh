# CG tile shapes at C2 (tasks must fit the SMs): per-iteration time at cap=100
cd /root/repo
for t in 3,4 3,3 3,2 2,4; do
  echo "tile $t"; CPKIT_CG_TILE=$t python tools/time_cg.py 2>&1 | grep "cap=  100"
done
