export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_p7.so
echo "p7 $(timeout 300 python -m pytest tests/test_gpu_2d.py -q -k "strip or full" 2>&1 | tail -1)"
for v in base p7 base p7; do
  if [ $v = base ]; then unset NMG_LIB; else export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so; fi
  echo "$v $(timeout 300 python tools/profile_cfg.py 3 256 2 | grep -E 'smooth' | tr '\n' ' ')"
done
