#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py (on the GPU box).
# Usage: bash tools/sanitize_all.sh <out-file> [case ...]
out=${1:-gpurun_out/sanitize.txt}; shift
: > "$out"
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize_cases.py $*" >> "$out"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py "$@" >> "$out" 2>&1
  echo "$tool rc=$?" >> "$out"
done
