#!/bin/bash
# Kernel-only bench for every build/ab/*.so under each environment setting:
#   tools/ab_matrix.sh "" "TTAGG_SERIAL=1" ...   (repeat passes with REPS=n)
cd "$(dirname "$0")/.."
for rep in $(seq ${REPS:-1}); do
  for so in build/ab/*.so; do
    n=$(basename $so .so)
    for envs in "$@"; do
      env $envs TTAGG_LIB=$PWD/$so python bench.py --no-cpu-baseline --no-e2e --rk2-steps 0 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$n [$envs]', round(d['ms_per_step'],3), {x:k[x] for x in k if k[x]>0.15})"
    done
  done
done
