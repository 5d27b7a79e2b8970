cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/r2o_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2o_pytest.txt
timeout 300 python tools/time_configs.py > gpurun_out/r2o_configs.txt 2>&1
CPKIT_SOLVE_ROWWISE=1 timeout 300 python tools/time_configs.py > gpurun_out/r2o_configs_rowwise.txt 2>&1
