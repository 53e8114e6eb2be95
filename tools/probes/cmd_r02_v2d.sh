mkdir -p gpurun_out
for w in c4ss c5ss; do
python tools/kernel_probe.py $w "" "EBIC_GAP=0" "EBIC_V2_SCHED=1" "EBIC_V2_SCHED=2" "EBIC_DEBUG_MODE=1" "EBIC_DEBUG_MODE=2" "EBIC_DEBUG_MODE=3" "EBIC_DEBUG_MODE=3 EBIC_V2_SCHED=1" "EBIC_DEBUG_MODE=3 EBIC_V2_SCHED=2" > gpurun_out/r02_v2d_$w.log 2>&1
done
EBIC_DEBUG_MODE=3 ncu --set full --clock-control none --import-source on -k regex:count_ -s 4 -c 1 -o gpurun_out/prof_r02_v2w3 python tools/kernel_probe.py c5ss > gpurun_out/ncu_r02_v2w3.log 2>&1
