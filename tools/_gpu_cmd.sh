timeout 900 python -m pytest tests -m gpu -q -x -k "coarse or cycle or smoke or history" 2>&1 | tail -1
for c in 0 1 2; do timeout 300 python tools/profile_cfg.py $c | grep -E "coarse" | tr '\n' ' '; echo; done
