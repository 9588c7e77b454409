#!/bin/bash
# A/B of libnmg variants on a config (default 3): ms/step and the smooth / filter class times.
# Usage: CFG=3 bash tools/ab_strip.sh [default|path/to/libnmg_X.so ...]   -- dev tool
cd "$(dirname "$0")/.."
for lib in ${@:-default}; do
  [ "$lib" = default ] && L= || L=$lib
  NMG_LIB=$L timeout 600 python bench.py --config ${CFG:-3} --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e --no-solve 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['classes_ms_per_step']; print('lib=$lib', round(d['ms_per_step'],3), ' '.join(f'{k} {v:.3f}' for k,v in r.items()), d['clocks']['sm_mhz'])"
done
