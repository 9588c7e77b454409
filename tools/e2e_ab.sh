#!/bin/bash
# e2e (host-buffer entry) vs device-entry throughput for nmg_tuning variants -- dev tool
# Usage: CFG=3 TUNES="default host_chunks=8" bash tools/e2e_ab.sh
cd "$(dirname "$0")/.."
for t in ${TUNES:-default host_chunks=8 host_chunks=12 host_chunks=16}; do
  [ "$t" = default ] && T= || T=$t
  timeout 600 python bench.py --config ${CFG:-3} --steps 3 --warmup 3 --no-cpu --no-solve ${T:+--tune $T} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tune=$t', round(d['ms_per_step'],1), round(d['value']), round(d['e2e']['value']), d['e2e']['check_vs_device_entry_max_rel_diff'])"
done
