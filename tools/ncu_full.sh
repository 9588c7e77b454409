#!/bin/bash
# One ncu --set full capture per hot kernel (run under gpurun, one GPU), after the same
# command has exited 0 without ncu.  Reports land in gpurun_out/ncu_<tag>.ncu-rep.
#   bash tools/ncu_full.sh [tags...]     (tags: s1d ozaki1d cfg3 cfg2 ... fno1 fno2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-solve"
run() {  # tag config kernel-regex count [extra bench args]
  timeout 900 $B --config $2 $5 > gpurun_out/plain_$1.log 2>&1 || { echo "PLAIN $1 failed"; return; }
  timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:$3" -c $4 \
      -o gpurun_out/ncu_$1 -f $B --config $2 $5 > gpurun_out/ncu_$1.log 2>&1
  echo "NCU $1 $?"
}
for t in ${@:-cfg3}; do
  case $t in
    s1d) run s1d 1 smooth1d_f16 1 "--lanes 1" ;;        # one lane: the full 1024-RHS launches
    ozaki1d) run ozaki1d 1 ozaki_resid 1 "--lanes 1" ;;
    cfg3) run cfg3 3 "conv_strip|fft_cols|fft_rows|combine_rows_fft|ozaki_resid|kron_tc|norms|sumsq" 14 ;;
    cfg2) run cfg2 2 "conv_strip|fft_cols|fft_rows|combine_rows_fft" 6 ;;
    strip3) run strip3 3 "conv_strip" 2 ;;
    strip2) run strip2 2 "conv_strip" 2 ;;
    fft3) run fft3 3 "fft_cols|fft_rows|combine_rows_fft|sumsq_partial" 4 "--lanes 1" ;;
    kron3) run kron3 3 "kron_tc" 4 ;;
    cols3) run cols3 3 "fft_cols|fft_rows" 2 "--lanes 1" ;;
    comb3) run comb3 3 "combine_rows" 1 "--lanes 1" ;;
    fno2) run fno2 2 "fno_conv_rows|fno_conv_tc|fno_rows_fwd|fno_rows_inv" 4 "--smoother fno --nrhs 64" ;;
    fno1) run fno1 1 "fno_conv_tc|fno_rows_fwd|fno_rows_inv" 3 "--smoother fno --nrhs 256 --lanes 1" ;;
  esac
done
