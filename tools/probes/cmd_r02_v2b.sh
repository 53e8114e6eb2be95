mkdir -p gpurun_out
for w in c4ss c5ss; do
python tools/kernel_probe.py $w "" "EBIC_V2_DYNAMIC=1" "EBIC_KERNEL=1" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" "EBIC_DEBUG_MODE=2 EBIC_V2_DYNAMIC=1" > gpurun_out/r02_v2b_$w.log 2>&1
done
