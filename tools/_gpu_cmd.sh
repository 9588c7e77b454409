timeout 600 python -m pytest tests/test_gpu_2d.py -q -x -k "ozaki or outer or history" 2>&1 | tail -2
for c in 2 4 3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ozaki|dgemm" --csv python tools/profile_cfg.py $c 32 1 2>/dev/null | grep -E "ozaki|dgemm" | awk -F'","' '{print $5, $NF}' | head -4
  NMG_FP64=dmma timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ozaki|dgemm" --csv python tools/profile_cfg.py $c 32 1 2>/dev/null | grep -E "ozaki|dgemm" | awk -F'","' '{print $5, $NF}' | head -2
done
