mkdir -p gpurun_out
for w in c4ss c5ss; do
python tools/kernel_probe.py $w "" "EBIC_COMPACT=1" "EBIC_COMPACT=0" "EBIC_KERNEL=1" "EBIC_COMPACT=1 EBIC_GAP=1" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" "EBIC_DEBUG_MODE=3" > gpurun_out/r02_v2e_$w.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02_v2e_parity.log 2>&1; echo EXIT $? >> gpurun_out/r02_v2e_parity.log
