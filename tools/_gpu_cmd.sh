timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for c in 1 2 4; do echo "$(timeout 300 python tools/profile_cfg.py $c | grep -E 'ms/step|transfer' | tr '\n' ' ')"; done
