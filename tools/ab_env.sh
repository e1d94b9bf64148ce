#!/bin/bash
# Kernel-only bench under several environment settings: tools/ab_env.sh "A=1 B=2" "A=2" ...
cd "$(dirname "$0")/.."
for envs in "$@"; do
  env $envs python bench.py --no-cpu-baseline --no-e2e --rk2-steps 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$envs', round(d['ms_per_step'],3), {x:k[x] for x in k if k[x]>0.15})"
done
