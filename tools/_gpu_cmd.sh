timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_strip" -c 2 -o gpurun_out/ncu_strip4 -f python tools/profile_cfg.py 2 256 1 > /dev/null 2>&1; echo "ncu2 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_strip" -c 2 -o gpurun_out/ncu_strip48 -f python tools/profile_cfg.py 3 64 1 > /dev/null 2>&1; echo "ncu3 $?"
