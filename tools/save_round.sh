#!/bin/bash
# copy the gpu_round.sh outputs into profiles/ (bench lines, ncu launch lists, per-kernel shares)
cd "$(dirname "$0")/.."
cp gpurun_out/bench_cfg1.json profiles/r01_bench.json
for c in 0 2 3 4; do cp gpurun_out/bench_cfg$c.json profiles/r01_bench_cfg$c.json; done
for c in 0 1 2 3 4; do
  cp gpurun_out/launches_cfg$c.csv profiles/r01_launches_cfg$c.csv
  python tools/launch_shares.py gpurun_out/launches_cfg$c.csv > profiles/r01_launch_shares_cfg$c.txt 2>/dev/null
done
cp gpurun_out/traffic.json profiles/traffic.json
