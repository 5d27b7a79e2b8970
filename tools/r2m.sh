cd /root/repo
CPKIT_ALLOC_TRACE=1 timeout 600 python tools/e2e_breakdown.py > gpurun_out/r2m_e2e.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2m_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r2m_pytest.txt
