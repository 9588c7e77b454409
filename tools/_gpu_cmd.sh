export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_g2p9.so
echo "g2p9 $(timeout 300 python -m pytest tests/test_gpu_2d.py -q -k strip 2>&1 | tail -1)"
for v in base g2p9 base g2p9; do
  if [ $v = base ]; then unset NMG_LIB; else export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so; fi
  for c in 2 4; do echo "$v $(timeout 300 python tools/profile_cfg.py $c | grep -E 'smooth' | tr '\n' ' ')"; done
done
