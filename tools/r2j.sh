cd /root/repo
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "spd or precond or gn_step or c1" > gpurun_out/r2j_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2j_pytest.txt
timeout 600 python tools/c5s_smoke.py > gpurun_out/r2j_c5s.txt 2>&1
CPKIT_CHOL_UNBLOCKED=1 timeout 600 python tools/c5s_smoke.py > gpurun_out/r2j_c5s_unblocked.txt 2>&1
