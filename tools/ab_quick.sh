#!/bin/bash
# Build, a focused GPU test subset, then interleaved kernel-only A/B runs of
# environment settings (REPS passes):  tools/ab_quick.sh TAG "A=0" "A=1" ...
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_dedup.py tests/test_gpu_guard.py} -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log; tail -3 gpurun_out/${TAG}_tests.log
for rep in $(seq ${REPS:-2}); do
  for envs in "$@"; do
    env $envs timeout 300 python bench.py --no-cpu-baseline --no-e2e --rk2-steps 0 ${BENCH_ARGS} 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('[$envs]', round(d['ms_per_step'],3), {x:k[x] for x in k if k[x]>0.15}, 'c4', round(d['c4_tt']['ms_per_rhs'],3) if d.get('c4_tt') else None)"
  done
done 2>&1 | tee gpurun_out/${TAG}_ab.log
[ -n "$EXTRA" ] && eval "$EXTRA"
exit 0
