cd /root/repo
for v in 0 1 2 4 8 7 15; do
  touch paper_1910_12331_b200/csrc/kernels_cg_res.cu
  make -s -C paper_1910_12331_b200/csrc EXTRA=-DCPKIT_CG_ABLATE=$v > /dev/null 2>&1 || echo build-fail
  echo "== ablate $v"
  CPKIT_CG_TILE=3,4 python tools/time_cg.py 2>&1 | tail -1
  CPKIT_CG_TILE=3,4 CPKIT_CG_TRACE=1 python tools/time_cg.py 2>&1 | grep "cg it" | tail -1
done
