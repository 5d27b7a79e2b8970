cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_full_configs.py -q -k "to_convergence" --durations=10 > gpurun_out/r2h_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.txt
