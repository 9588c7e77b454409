timeout 900 ncu --set full --clock-control none --import-source on -k regex:kron_tc --launch-skip 3 -c 1 -o gpurun_out/ncu_kron1 -f python tools/profile_cfg.py 4 32 1 > /dev/null 2>&1; echo "ncu $?"
