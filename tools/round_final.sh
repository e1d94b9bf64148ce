#!/bin/bash
# Round-end validation on one GPU: smoke, GPU tests, default bench line, the
# reference arm, ncu launch list and a full ncu capture of one C5 RHS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
bash tools/round_profile.sh
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench_ref.log | cut -c1-400
