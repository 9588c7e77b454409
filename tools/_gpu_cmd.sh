timeout 600 python -m pytest tests/test_gpu_1d.py -q -x 2>&1 | tail -1
for lt in 1 0 1 0; do
  echo "lane_tiles $lt: $(NMG_LANE_TILES=$lt timeout 300 python bench.py --config 1 --steps 100 --no-cpu --no-e2e --no-solve | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"
done
