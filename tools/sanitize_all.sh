#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_case.py
# (CP d=3..5 + TT d=2 RHS and 3 fused RK2 steps); logs to gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-4096}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py $N \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.log
done
# the N1 = 4096 geometry (TMA pass A / pass B kernels) under memcheck
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py 1048576 \
  > gpurun_out/sanitize_memcheck_2p20.log 2>&1
echo "exit=$?" >> gpurun_out/sanitize_memcheck_2p20.log
