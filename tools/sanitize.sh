#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (one small launch of every kernel path)
# -> gpurun_out/sanitizer/{memcheck,racecheck,synccheck,initcheck,memcheck_exact_alloc}.txt
mkdir -p gpurun_out/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitizer/$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/$tool.txt
done
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 $S --tool memcheck --error-exitcode 9 python tools/sanitize_case.py \
  > gpurun_out/sanitizer/memcheck_exact_alloc.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/memcheck_exact_alloc.txt
