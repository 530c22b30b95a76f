#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (one GPU); summaries to gpurun_out/<tag>/
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
SAN_GRAPH=1 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > $OUT/memcheck_graph.log 2>&1
echo "memcheck(graph) rc=$? $(grep -E 'ERROR SUMMARY' $OUT/memcheck_graph.log | tail -1)"
