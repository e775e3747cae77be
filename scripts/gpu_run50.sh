# compute-sanitizer on the small end-to-end runs after this session's kernel changes.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py > gpurun_out/r50_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r50_sanitizer_$tool.txt
done
