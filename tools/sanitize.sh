# compute-sanitizer evidence (SURVEY §5 / VERDICT r01): memcheck, racecheck,
# synccheck and initcheck over tools/sanitize_driver.py, which drives every
# kernel family (TMA + mbarrier root GEMM, cooperative CG with the software grid
# barrier, cluster/DSMEM Gram, blocked Cholesky, graphs, tiny instances).
# Usage (GPU box): bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out}
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, label, extra env
  local tool=$1 label=$2; shift 2
  env "$@" timeout 1500 $CS --tool $tool --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_driver.py > $OUT/san_${label}.txt 2>&1
  echo "$label rc=$?" | tee -a $OUT/san_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|Error|ok|done" $OUT/san_${label}.txt | tail -4 >> $OUT/san_summary.txt
}
: > $OUT/san_summary.txt
run memcheck memcheck
run memcheck memcheck_alt CPKIT_CG_STREAMING=1 CPKIT_ALS_TREE=1 CPKIT_CHOL_UNBLOCKED=1 CPKIT_GN_SYNC=1 CPKIT_NO_GRAPH=1
run synccheck synccheck SAN_SMALL=1
run initcheck initcheck SAN_SMALL=1
run racecheck racecheck SAN_SMALL=1
run racecheck racecheck_alt SAN_SMALL=1 CPKIT_CG_STREAMING=1 CPKIT_CHOL_UNBLOCKED=1
cat $OUT/san_summary.txt
