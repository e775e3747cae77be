#!/usr/bin/env bash
# compute-sanitizer tools over scripts/sanitize_small.py; one summary line per tool (+ racecheck hazard sites)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
O=gpurun_out/${1:-san}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  [ "$tool" = racecheck ] && export MGGCN_RACECHECK=1 || unset MGGCN_RACECHECK
  timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_small.py > ${O}_$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' ${O}_$tool.log | tail -1)"
  grep -E "access at" ${O}_$tool.log | sed 's/0x[0-9a-f]*//g' | sort | uniq -c | sort -rn | head -5
done
