# Full measurement pass (GPU box): bench (ours + reference arm), the bench's
# launch list (ncu duration pass of the same command), the CG kernel timings,
# the C2 ALS/GN CUPTI timelines and smoke().
cd /root/repo
OUT=${1:-gpurun_out/measure}
mkdir -p $OUT
set -x
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
python tools/launch_summary.py $OUT/launches_bench.csv > $OUT/launches_summary.txt
REPEAT=2 timeout 300 python tools/time_cg.py > $OUT/time_cg_c2.txt 2>&1
timeout 300 python tools/timeline_als.py > $OUT/timeline_als.txt 2>&1
timeout 300 python tools/timeline_als.py gn > $OUT/timeline_gn.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
tail -c 600 $OUT/bench.json
tail -1 $OUT/smoke.log
