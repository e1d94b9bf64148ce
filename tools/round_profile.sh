#!/bin/bash
# One GPU session: GPU tests, the default bench line, the ncu launch list of a
# short bench run and a full ncu capture of one C5 RHS (outputs in gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --rk2-steps 0 --no-c4 > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --launch-skip 18 --launch-count 18 \
  -o gpurun_out/rhs_full -f python tools/prof_rhs.py 1048576 2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -2 gpurun_out/bench.log | cut -c1-300; ls gpurun_out
