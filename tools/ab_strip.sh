#!/bin/bash
# A/B of conv_strip variants on config 3 (smooth class per step) -- dev tool
cd "$(dirname "$0")/.."
for lib in "" ${@}; do
  NMG_LIB=$lib timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-solve 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['classes_ms_per_step']; print('lib=${lib:-default}', round(d['ms_per_step'],2), 'smooth', round(r['smooth'],2), 'filter', round(r['filter'],2), d['clocks']['sm_mhz'])"
done
