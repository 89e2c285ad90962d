#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py -> gpurun_out/<tag>_san_*.txt
cd "$(dirname "$0")/.."
tag=${1:-san}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 7 python tools/sanitize.py > gpurun_out/${tag}_san_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/${tag}_san_$tool.txt
  tail -4 gpurun_out/${tag}_san_$tool.txt
done
