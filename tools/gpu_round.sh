#!/bin/bash
# One GPU-box pass: build, GPU tests, smoke, default bench, sharded bench at 1 GPU.
# usage: bash tools/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_sharded.log 2>&1
