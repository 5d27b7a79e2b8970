cd /root/repo
timeout 600 python -m pytest tests/test_gpu_cg_cluster.py -q -x > gpurun_out/r2f_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2f_pytest.txt
CPKIT_CG_TRACE=1 timeout 300 python tools/profile_cg.py > gpurun_out/r2f_cg_trace.txt 2>&1
for v in "" "CPKIT_CG_HIER=1" "CPKIT_CG_NO_CLUSTER=1"; do
  echo "== $v" >> gpurun_out/r2f_time_cg.txt
  env $v REPEAT=2 timeout 300 python tools/time_cg.py >> gpurun_out/r2f_time_cg.txt 2>&1
done
