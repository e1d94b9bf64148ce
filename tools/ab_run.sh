#!/bin/bash
# Run the kernel-only bench for each build/ab/*.so: prints name, ms/RHS, per-kernel ms.
cd "$(dirname "$0")/.."
for so in build/ab/*.so; do
  n=$(basename $so .so)
  TTAGG_LIB=$PWD/$so python bench.py --no-cpu-baseline --no-e2e --rk2-steps 0 "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$n', round(d['ms_per_step'],3), {x:k[x] for x in k if k[x]>0.15})"
done
