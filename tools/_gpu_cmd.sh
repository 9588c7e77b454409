timeout 600 python -m pytest tests/test_gpu_1d.py -q -x 2>&1 | tail -1
for ln in 2 1 2 1; do
  if [ $ln = 1 ]; then export NMG_LANES=1; else unset NMG_LANES; fi
  echo "lanes $ln: $(timeout 300 python bench.py --config 1 --steps 100 --no-cpu --no-e2e --no-solve | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"
done
