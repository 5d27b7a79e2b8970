cd /root/repo
for v in "" "CPKIT_NN_NT8=5 CPKIT_NN_WM=8 CPKIT_NN_NW=8" "CPKIT_NN_NT8=5 CPKIT_NN_WM=10 CPKIT_NN_NW=10" "CPKIT_NN_NT8=5 CPKIT_NN_WM=4 CPKIT_NN_NW=4" "CPKIT_NN_NT8=5 CPKIT_NN_WM=8 CPKIT_NN_NW=8 CPKIT_NN_STAGES=4"; do
  echo "== $v" >> gpurun_out/r2n.txt
  env $v CPKIT_PLAN_DEBUG=1 timeout 300 python tools/c5s_smoke.py >> gpurun_out/r2n.txt 2>&1
done
