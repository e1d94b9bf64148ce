#!/bin/bash
# One GPU session: GPU tests, the default bench line, the ncu launch list of a
# short bench run and a full ncu capture of one C5 RHS (outputs in gpurun_out/).
# usage: bash tools/round_profile.sh [TAG]
cd "$(dirname "$0")/.."
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --rk2-steps 0 --no-c4 --no-extras > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 18 --launch-count 18 \
  -o gpurun_out/${TAG}_rhs_full -f python tools/prof_rhs.py 1048576 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -2 gpurun_out/${TAG}_gpu_tests.log; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300; ls gpurun_out
