# CG cost attribution: per-iteration time with parts of the iteration disabled
# (CPKIT_CG_ABLATE bits, kernels_cg_res.cu: 1 A2 work, 2 gathers, 4 GEMMs,
# 8 slot sums, 16 phase-A publish; numerically wrong, timing only).
cd /root/repo
for v in ${ABLATE:-0 1 2 4 8 12 13}; do
  touch paper_1910_12331_b200/csrc/kernels_cg_res.cu
  make -s -C paper_1910_12331_b200/csrc EXTRA=-DCPKIT_CG_ABLATE=$v > /dev/null 2>&1 || echo build-fail
  echo "== ablate $v"
  python tools/time_cg.py 2>&1 | tail -1
  CPKIT_CG_TRACE=1 python tools/cg_trace.py 2>&1 | grep "cg it 2[0-1]"
done
touch paper_1910_12331_b200/csrc/kernels_cg_res.cu
make -s -C paper_1910_12331_b200/csrc > /dev/null 2>&1
