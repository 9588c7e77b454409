#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench lines for the configs, per-rank shard timings (the
# strong-scaling prediction), and ncu launch lists with DRAM bytes for the configs' steps
# (merged into gpurun_out/traffic.json).  Usage (under gpurun): bash tools/gpu_round.sh [configs...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${@:-"3 1 0 2 4"}
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/gputests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/smoke.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "BENCH $c $?"
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));print(d['ms_per_step'], d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['frac'], d.get('solve'))"
done
if [ -n "$SHARDS" ]; then
  # per-GPU shard of an 8-GPU split (strong scaling): T(B) vs T(B/8)
  for spec in 1:128 2:32 3:256; do
    c=${spec%%:*}; b=${spec#*:}
    timeout 600 python bench.py --config $c --nrhs $b --no-cpu --no-e2e --no-solve > gpurun_out/shard_cfg$c.json 2>/dev/null
    echo "SHARD $c $b $(python -c "import json;d=json.load(open('gpurun_out/shard_cfg$c.json'));print(d['ms_per_step'])")"
  done
fi
if [ -n "$NCU" ]; then
  cp profiles/traffic.json gpurun_out/traffic.json 2>/dev/null
  for c in $NCU; do
    L=$(python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));print(int(round(sum(d['roofline']['launches_per_step'].values()))))")
    CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e --no-solve"
    timeout 600 $CMD > gpurun_out/plain_cfg$c.log 2>&1 && \
    timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_cfg$c.log 2>&1
    echo "NCU $c $? (launches/step $L)"
    python tools/ncu_traffic.py gpurun_out/launches_cfg$c.csv $L gpurun_out/traffic.json cfg$c
  done
fi
