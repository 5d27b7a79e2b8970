cd /root/repo
timeout 900 python -m pytest tests/test_gpu_guard.py "tests/test_gpu_configs.py::test_gn_reference_residual_semantics" -q > gpurun_out/r2c_pytest_new.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c_pytest_new.txt
CPKIT_CG_TRACE=1 timeout 300 python tools/profile_cg.py > gpurun_out/r2c_cg_trace.txt 2>&1
CPKIT_CG_TRACE=1 timeout 300 python tools/profile_cg.py 200,200,200 20 > gpurun_out/r2c_cg_trace_c3.txt 2>&1
CPKIT_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2c_pytest_guard.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c_pytest_guard.txt
tail -3 gpurun_out/r2c_pytest_new.txt gpurun_out/r2c_pytest_guard.txt
