cd /root/repo
CPKIT_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest_guard.txt 2>&1
echo "rc=$?" >> gpurun_out/r2d_pytest_guard.txt
CPKIT_PLAN_DEBUG=1 timeout 300 python tools/profile_roots.py 200,200,200,200 200 > gpurun_out/r2d_plan_c5s.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:root_gemm_kernel -c 2 \
    -o gpurun_out/r2d_roots_c5s python tools/profile_roots.py 200,200,200,200 200 > gpurun_out/r2d_ncu_c5s.log 2>&1
tail -3 gpurun_out/r2d_pytest_guard.txt
