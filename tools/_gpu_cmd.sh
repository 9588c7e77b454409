timeout 600 python -m pytest tests/test_gpu_1d.py -q -x 2>&1 | tail -1
for mc in 1 0; do NMG_GEMM_MC=$mc timeout 300 python tools/profile_cfg.py 1 1024 20 | grep -E "ms/step|gemm32"; done
for mc in 1 0; do NMG_GEMM_MC=$mc timeout 300 python tools/profile_cfg.py 1 1024 20 | grep -E "ms/step|gemm32"; done
