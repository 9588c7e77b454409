#!/bin/bash
# Zero-block K skipping A/B: bitwise-equality and scale-regime tests, then configs 1 and 3 (and 2)
# with the default path and with nmg_tuning.dense_k = 1 (every K block).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kskip.py tests/test_gpu_scale_regime.py -q -x > gpurun_out/tkskip.log 2>&1; echo "TKSKIP $?"; tail -3 gpurun_out/tkskip.log
for c in ${CFGS:-1 3 2}; do
  for t in "" "dense_k=1"; do
    timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e --no-solve --tune "$t" 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['classes_ms_per_step']; print('tune=$t cfg$c', round(d['ms_per_step'],4), {k: round(v,3) for k,v in r.items()}, d['clocks']['sm_mhz'])"
  done
done
