#!/bin/bash
# 1D A/B: parity tests of the 1D path, then config 1 (full batch and a 128-RHS shard) and config 0
# with the fused coarse sub-cycle on / off.
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_1d.py tests/test_gpu_variants.py -q -x > gpurun_out/t1d.log 2>&1; echo "T1D $?"; tail -2 gpurun_out/t1d.log
timeout 900 python -m pytest tests/test_gpu_launch_configs.py -q -x -k "cfg1" > gpurun_out/tlc.log 2>&1; echo "TLC $?"; tail -2 gpurun_out/tlc.log
for t in "" "no_fused_coarse=1"; do
  for spec in "1:0" "1:128" "0:0"; do
    c=${spec%%:*}; b=${spec#*:}; nr=""; [ "$b" != "0" ] && nr="--nrhs $b"
    timeout 600 python bench.py --config $c $nr --steps ${STEPS:-200} --warmup 5 --no-cpu --no-e2e --no-solve --tune "$t" 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['classes_ms_per_step']; print('tune=$t cfg$c nrhs=$b', round(d['ms_per_step'],4), {k: round(v,3) for k,v in r.items()})"
  done
done
