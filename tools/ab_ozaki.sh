#!/bin/bash
# A/B of the Ozaki fp64 residual pipeline (default build vs variants/libnmg_oz64.so): parity tests
# of the fp64 residual, then the gemm64 class time per step for configs 1 and 3.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q -x -k "outer_residual or residual_2d or slab or wseed_alpha or tiled_pool or history" > gpurun_out/oz_tests.log 2>&1; echo "OZTESTS $?"; tail -2 gpurun_out/oz_tests.log
for lib in "" paper_2603_01064_b200/variants/libnmg_oz64.so; do
  for c in 1 3; do
    NMG_LIB=$lib timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e --no-solve 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['classes_ms_per_step']; print('lib=${lib:-default} cfg$c', round(d['ms_per_step'],3), 'gemm64', round(r['gemm64'],3), d['clocks']['sm_mhz'])"
  done
done
