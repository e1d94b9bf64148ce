#!/bin/bash
# Interleaved kernel-only bench of build/ab/*.so (REPS passes): C5 ms/RHS, pass A/B d=5, and the D=4 / C3 / C4 lines.
cd "$(dirname "$0")/.."
for rep in $(seq ${REPS:-2}); do
for so in build/ab/*.so; do
  n=$(basename $so .so)
  TTAGG_LIB=$PWD/$so timeout 600 python bench.py --no-cpu-baseline --no-e2e --rk2-steps 0 "$@" 2>/dev/null | tail -1 | \
    python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; e=d.get('extras') or {}
print('$n', 'rhs', round(d['ms_per_step'],3), 'A5', k.get('A5'), 'B5', k.get('B5'), 'A4', k.get('A4'),
      'd4', round(e['d4_n2p20']['ms_per_rhs'],3) if 'd4_n2p20' in e else None,
      'c3', round(e['c3']['ms_per_rhs'],4) if 'c3' in e else None,
      'c4', round(d['c4_tt']['ms_per_rhs'],3) if d.get('c4_tt') else None, 'mhz', d.get('clocks',{}).get('sm_mhz'))"
done
done
