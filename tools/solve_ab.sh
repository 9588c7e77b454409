#!/bin/bash
# A/B of the solve figure (RHS solved to 1e-6 per second) across libnmg variants -- dev tool
# Usage: CFG=3 bash tools/solve_ab.sh [default|path/to/libnmg_X.so ...]
cd "$(dirname "$0")/.."
for lib in ${@:-default}; do
  [ "$lib" = default ] && L= || L=$lib
  NMG_LIB=$L timeout 900 python bench.py --config ${CFG:-3} --steps 2 --warmup 3 --no-cpu --no-e2e ${TUNE:+--tune $TUNE} 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print('lib=$lib', round(s['value'],1), s['cycles_max'], s['cycles_mean'], round(s['seconds'],3), s['converged'])"
done
