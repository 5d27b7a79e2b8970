cd /root/repo
for v in 0 1 2 4 7; do
  touch paper_1910_12331_b200/csrc/kernels_chol.cu
  make -s -C paper_1910_12331_b200/csrc EXTRA=-DCPKIT_CHOL_ABLATE=$v > /dev/null 2>&1 || echo build-fail
  echo "== ablate $v"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:chol_blocked python tools/time_spd.py 2>/dev/null | grep -E "chol" | awk -F, '{print $(NF)}' | tr '\n' ' '; echo
done
