#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench lines for configs 0-4, and per-config ncu launch
# lists with DRAM bytes (merged into gpurun_out/traffic.json).  Usage (under gpurun):
#   bash tools/gpu_round.sh [configs...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${@:-"1 0 2 3 4"}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "SMOKE $?"
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "BENCH $c $?"
done
cp profiles/traffic.json gpurun_out/traffic.json 2>/dev/null
for c in $CFGS; do
  L=$(python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));print(int(round(sum(d['roofline']['launches_per_step'].values()))))")
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e --no-solve"
  timeout 600 $CMD > gpurun_out/plain_cfg$c.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_cfg$c.log 2>&1
  echo "NCU $c $? (launches/step $L)"
  python tools/ncu_traffic.py gpurun_out/launches_cfg$c.csv $L gpurun_out/traffic.json cfg$c
done
