#!/bin/bash
# copy the gpu_round.sh outputs into profiles/ (bench lines, ncu launch lists, per-kernel shares)
# Usage: bash tools/save_round.sh [round tag, default r02]
cd "$(dirname "$0")/.."
R=${1:-r02}
for c in 0 1 2 3 4; do
  [ -s gpurun_out/bench_cfg$c.json ] && cp gpurun_out/bench_cfg$c.json profiles/${R}_bench_cfg$c.json
  [ -s gpurun_out/shard_cfg$c.json ] && cp gpurun_out/shard_cfg$c.json profiles/${R}_shard_cfg$c.json
  if [ -s gpurun_out/launches_cfg$c.csv ]; then
    cp gpurun_out/launches_cfg$c.csv profiles/${R}_launches_cfg$c.csv
    python tools/launch_shares.py gpurun_out/launches_cfg$c.csv > profiles/${R}_launch_shares_cfg$c.txt 2>/dev/null
  fi
done
[ -s gpurun_out/traffic.json ] && cp gpurun_out/traffic.json profiles/traffic.json
