export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_tw.so
echo "tw $(timeout 300 python -m pytest tests/test_gpu_1d.py -q 2>&1 | tail -1)"
for v in base tw base tw; do
  if [ $v = base ]; then unset NMG_LIB; else export NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_$v.so; fi
  echo "$v: $(timeout 300 python bench.py --config 1 --steps 100 --no-cpu --no-e2e --no-solve | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["classes_ms_per_step"]["smooth"])')"
done
NMG_LANES=1 NMG_GRAPH=0 NMG_LIB=$PWD/paper_2603_01064_b200/variants/libnmg_twph.so timeout 300 python tools/profile_cfg.py 1 1024 1 2>&1 | grep s1d | sort -k2 | awk 'NR%3==1'
