# CG gather cost: baseline vs copy_rows disabled (ablate 2; numerically wrong, timing only)
cd /root/repo
for v in 0 2; do
  touch paper_1910_12331_b200/csrc/kernels_cg_res.cu
  make -s -C paper_1910_12331_b200/csrc EXTRA=-DCPKIT_CG_ABLATE=$v > /dev/null 2>&1 || echo build-fail
  echo "== ablate $v"
  CPKIT_CG_TRACE=1 python tools/time_cg.py 2>&1 | grep "cg it 2[0-1]"
done
touch paper_1910_12331_b200/csrc/kernels_cg_res.cu
make -s -C paper_1910_12331_b200/csrc > /dev/null 2>&1
