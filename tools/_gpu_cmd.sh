timeout 600 python -m pytest tests/test_gpu_1d.py -q -x -k "lanes or cycle" 2>&1 | tail -1
for ln in 2 3 4 2 3 4; do echo "lanes $ln: $(NMG_LANES=$ln timeout 300 python bench.py --config 1 --steps 100 --no-cpu --no-e2e --no-solve | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"; done
