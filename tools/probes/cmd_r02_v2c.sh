mkdir -p gpurun_out
for w in c4ss c5ss; do
python tools/kernel_probe.py $w "" "EBIC_GAP=0" "EBIC_GAP=1" "EBIC_V2_SCHED=1" "EBIC_V2_SCHED=2" "EBIC_KERNEL=1" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" > gpurun_out/r02_v2c_$w.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02_v2c_parity.log 2>&1; echo EXIT $? >> gpurun_out/r02_v2c_parity.log
