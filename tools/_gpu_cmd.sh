timeout 600 python -m pytest tests/test_gpu_1d.py -q -x 2>&1 | tail -1
for v in base m5 base m5; do
  if [ $v = base ]; then unset NMG_LIB; else export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so; fi
  echo "$v: $(timeout 300 python bench.py --config 1 --steps 100 --no-cpu --no-e2e --no-solve | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["classes_ms_per_step"]["smooth"])')"
done
