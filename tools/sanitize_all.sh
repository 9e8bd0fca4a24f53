# compute-sanitizer over tools/sanitize_small.py (every entry point, incl. the TMA-staged stream);
# racecheck once more with SANITIZE_NO_BULK=1 (per-thread weight loads) as the control
CS=/usr/local/cuda/bin/compute-sanitizer
# synccheck runs the kgen_bal barriers in their synccheck-clean form (FDIRW_KGEN_SYNCCHECK=1, the
# same barrier sequence through one non-inlined call; kgen_common.cuh): synccheck expects one PC per
# CTA barrier and reports the default named-barrier form of the warp-specialised segments
for tool in memcheck racecheck synccheck initcheck; do
  SC=0; [ $tool = synccheck ] && SC=1
  FDIRW_KGEN_SYNCCHECK=$SC timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(tail -2 gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
SANITIZE_NO_BULK=1 timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_racecheck_nobulk.log 2>&1
echo "racecheck (no bulk) rc=$? $(tail -2 gpurun_out/sanitize_racecheck_nobulk.log | tr '\n' ' ')"
