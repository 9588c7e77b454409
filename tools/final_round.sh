#!/bin/bash
# Round-end GPU pass: gpu_round.sh (tests, smoke, CNN bench lines, shard timings, ncu launch lists)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SHARDS=1 NCU="3 1" bash tools/gpu_round.sh 3 1 0 2 4
for c in 0 1 2; do
  timeout 900 python bench.py --config $c --smoother fno > gpurun_out/bench_fno_cfg$c.json 2> gpurun_out/bench_fno_cfg$c.err; echo "BENCH fno $c $?"
  python -c "import json;d=json.load(open('gpurun_out/bench_fno_cfg$c.json'));print(d['ms_per_step'], d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['frac'])"
done
timeout 900 python bench.py --config 3 --smoother fno --nrhs 64 --no-cpu > gpurun_out/bench_fno_cfg3_64.json 2> gpurun_out/bench_fno_cfg3_64.err; echo "BENCH fno 3/64 $?"
for spec in 1:256 2:64; do
  c=${spec%%:*}; b=${spec#*:}
  CMD="python bench.py --config $c --smoother fno --steps 1 --warmup 1 --no-cpu --no-e2e --nrhs $b"
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches_fno_cfg$c.csv $CMD > gpurun_out/ncu_fno_cfg$c.log 2>&1; echo "NCU fno $c $?"
done
