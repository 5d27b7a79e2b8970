# round-2 GPU pass: full gpu suite, sanitizers, ncu of the current CG kernel
cd /root/repo
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2b_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cg_res_kernel -c 1 \
    -o gpurun_out/r2b_cg_full python tools/profile_cg.py > gpurun_out/r2b_ncu_cg.log 2>&1
timeout 2400 bash tools/sanitize.sh gpurun_out > gpurun_out/r2b_san.log 2>&1
tail -3 gpurun_out/r2b_pytest.txt
