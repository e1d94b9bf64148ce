#!/bin/bash
# One GPU-box pass: build, GPU tests, smoke, default bench, sharded bench at 1 GPU,
# and a timing of one whole CPU RHS (the reference arm's unit of work).
# usage: bash tools/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/${TAG}_host.txt; free -g >> gpurun_out/${TAG}_host.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_sharded.log 2>&1
[ -n "$CPU_PROBE" ] && timeout 600 python tools/cpu_rhs_probe.py 16 > gpurun_out/${TAG}_cpuprobe.log 2>&1
exit 0
