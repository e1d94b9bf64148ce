#!/bin/bash
# C4-shape TT timing (tools/bench_tt.py) for every build/ab/*.so: tools/ab_tt.sh [rank]
cd "$(dirname "$0")/.."
for rep in $(seq ${REPS:-1}); do
  for so in build/ab/*.so; do
    echo -n "$(basename $so .so) "; TTAGG_LIB=$PWD/$so python tools/bench_tt.py ${1:-16} 2>/dev/null | tail -1
  done
done
