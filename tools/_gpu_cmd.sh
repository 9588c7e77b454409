timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_2d.py tests/test_gpu_1d.py -q -x 2>&1 | tail -1
for v in base old base old; do
  if [ $v = base ]; then unset NMG_LIB; else export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so; fi
  echo "$v $(timeout 300 python tools/profile_cfg.py 4 | grep -E 'gemm64' | tr '\n' ' ')"
done
