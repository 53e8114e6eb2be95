mkdir -p gpurun_out
EBIC_DEBUG_MODE=2 ncu --set full --clock-control none --import-source on -k regex:count_ -s 4 -c 1 -o gpurun_out/prof_r02_v2walk python tools/kernel_probe.py c5ss > gpurun_out/ncu_r02_v2walk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:count_ -s 4 -c 1 -o gpurun_out/prof_r02_v2c5 python tools/kernel_probe.py c5ss > gpurun_out/ncu_r02_v2c5.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_r02_v2c5.log
