mkdir -p gpurun_out
python tools/kernel_probe.py c4ss "" "EBIC_KERNEL=1" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" > gpurun_out/r02_v2_c4ss.log 2>&1
python tools/kernel_probe.py c5ss "" "EBIC_KERNEL=1" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" > gpurun_out/r02_v2_c5ss.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02_v2_parity.log 2>&1; echo EXIT $? >> gpurun_out/r02_v2_parity.log
