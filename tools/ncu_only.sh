#!/bin/bash
# ncu launch list of a short bench run + full capture of one C5 RHS (no tests, no bench line).
# usage: bash tools/ncu_only.sh TAG
cd "$(dirname "$0")/.."
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --rk2-steps 0 --no-c4 --no-extras > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 18 --launch-count 18 \
  -o gpurun_out/${TAG}_rhs_full -f python tools/prof_rhs.py 1048576 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out | tail -5
