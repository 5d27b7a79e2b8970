# Full measurement pass (GPU box): bench (ours + reference arm), launch list, ncu capture of the roots.
cd /root/repo
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/profile_roots.py > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:root_gemm_kernel -c 2 \
    -o gpurun_out/roots_full python tools/profile_roots.py > gpurun_out/ncu_roots.log 2>&1
python tools/profile_cg.py > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:cg_res_kernel -c 1 \
    -o gpurun_out/cg_full python tools/profile_cg.py > gpurun_out/ncu_cg.log 2>&1
tail -c 600 gpurun_out/bench.json
python tools/profile_tiny.py gn > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:tiny_kernel -c 1 \
    -o gpurun_out/tiny_full python tools/profile_tiny.py gn > gpurun_out/ncu_tiny.log 2>&1
python tools/bench_likelihood.py gn > gpurun_out/likelihood.txt 2>&1
python tools/bench_likelihood.py als >> gpurun_out/likelihood.txt 2>&1
