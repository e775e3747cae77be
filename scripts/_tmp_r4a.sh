cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_run.sh r4a suite bench
grep -E "^FAILED|passed|failed" gpurun_out/r4a_pytest.log | tail -5
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_small.py > gpurun_out/r4a_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/r4a_$tool.log | head -2; grep -E "hazards\]" gpurun_out/r4a_$tool.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | cut -c1-160 | head -4
done
