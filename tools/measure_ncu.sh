# ncu --set full captures of the dominant kernels (one GPU): the C5s and C2 root
# GEMMs (tools/profile_roots.py) and the tile-resident CG at C2 in its gather
# variant (ncu cannot replay the cluster-mode cooperative launch).
cd /root/repo
OUT=${1:-gpurun_out/ncu}
mkdir -p $OUT
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:root_gemm -c 6 -f -o $OUT/roots_c5s \
    python tools/profile_roots.py 200,200,200,200 200 > $OUT/roots_c5s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:root_gemm -c 12 -f -o $OUT/roots_c2 \
    python tools/profile_roots.py > $OUT/roots_c2.log 2>&1
CPKIT_CG_NO_CLUSTER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_res -c 1 -f \
    -o $OUT/cg_c2 python tools/profile_cg.py > $OUT/cg_c2.log 2>&1
ls -la $OUT
# summaries are made on the box (the reports exceed the 64 MiB gpurun_out limit)
python tools/ncu_summary.py $OUT/roots_c5s.ncu-rep > $OUT/ncu_roots_c5s_summary.txt 2>&1
python tools/make_ncu_summary.py $OUT/roots_c5s.ncu-rep $OUT/ncu_roots_c5s.json "tools/profile_roots.py 200,200,200,200 200 (C5s roots)" > /dev/null 2>&1
python tools/ncu_summary.py $OUT/roots_c2.ncu-rep > $OUT/ncu_roots_c2_summary.txt 2>&1
python tools/make_ncu_summary.py $OUT/roots_c2.ncu-rep $OUT/ncu_roots_c2.json "tools/profile_roots.py (C2 roots)" > /dev/null 2>&1
python tools/ncu_summary.py $OUT/cg_c2.ncu-rep 12 > $OUT/ncu_cg_summary.txt 2>&1
python tools/ncu_lines.py $OUT/cg_c2.ncu-rep > $OUT/ncu_cg_lines.txt 2>&1
rm -f $OUT/*.ncu-rep
