for v in s5 s6 s7 s8; do
  export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so
  echo "== $v $(timeout 300 python -m pytest tests/test_gpu_2d.py -q -k strip 2>&1 | tail -1)"
  for c in 2 4; do timeout 300 python tools/profile_cfg.py $c | grep -E "ms/step|smooth"; done
done
