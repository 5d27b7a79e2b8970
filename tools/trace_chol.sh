# Cholesky phase trace (CTA 0 globaltimer stamps): rebuild with CPKIT_CHOL_TRACE, run
# the SPD driver and a few eager ALS sweeps, rebuild normally.
cd /root/repo
touch paper_1910_12331_b200/csrc/kernels_chol.cu
make -s -C paper_1910_12331_b200/csrc EXTRA=-DCPKIT_CHOL_TRACE=1 > /dev/null 2>&1 || echo build-fail
python tools/time_spd.py 2>&1 | grep "chol" | head -4
CPKIT_NO_GRAPH=1 SWEEPS=2 python tools/profile_als.py 2>&1 | grep "chol" | tail -2
touch paper_1910_12331_b200/csrc/kernels_chol.cu
make -s -C paper_1910_12331_b200/csrc > /dev/null 2>&1
