timeout 1200 python -m pytest tests/test_gpu_2d.py tests/test_gpu_slab.py tests/test_gpu_variants.py -q -x 2>&1 | tail -1
for c in 2 4; do echo "$(timeout 300 python tools/profile_cfg.py $c | grep -E 'ms/step|smooth' | tr '\n' ' ')"; done
