export AIRG_GM_FLAT=1 AIRG_DEVLOOP=0
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"
  tail -3 gpurun_out/san_$t.log
done
