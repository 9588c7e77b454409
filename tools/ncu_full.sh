#!/bin/bash
# One ncu --set full capture per hot kernel (run under gpurun, one GPU), after the same
# command has exited 0 without ncu.  Reports land in gpurun_out/ncu_<tag>.ncu-rep.
#   bash tools/ncu_full.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-solve"
run() {  # tag config kernel-regex count
  timeout 600 $B --config $2 > gpurun_out/plain_$1.log 2>&1 || { echo "PLAIN $1 failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -c $4 \
      -o gpurun_out/ncu_$1 -f $B --config $2 > gpurun_out/ncu_$1.log 2>&1
  echo "NCU $1 $?"
}
NMG_LANES=1 run s1d 1 smooth1d_f16 1     # one lane: the full 1024-RHS launches
NMG_LANES=1 run ozaki 1 ozaki_resid 1
run strip2 2 "conv_strip|fft_cols|fft_rows" 4
