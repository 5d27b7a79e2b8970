cd /root/repo
timeout 600 python -m pytest tests/test_gpu_cg_cluster.py -q -x > gpurun_out/r2e_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2e_pytest.txt
CPKIT_CG_TRACE=1 timeout 300 python tools/profile_cg.py > gpurun_out/r2e_cg_trace.txt 2>&1
CPKIT_CG_TRACE=1 CPKIT_CG_NO_CLUSTER=1 timeout 300 python tools/profile_cg.py > gpurun_out/r2e_cg_trace_gather.txt 2>&1
REPEAT=3 timeout 300 python tools/time_cg.py > gpurun_out/r2e_time_cg.txt 2>&1
CPKIT_CG_NO_CLUSTER=1 REPEAT=3 timeout 300 python tools/time_cg.py > gpurun_out/r2e_time_cg_gather.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_pytest_all.txt 2>&1
echo "rc=$?" >> gpurun_out/r2e_pytest_all.txt
