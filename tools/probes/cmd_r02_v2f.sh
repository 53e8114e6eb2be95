mkdir -p gpurun_out
for w in c4ss c5ss; do
python tools/kernel_probe.py $w "" "EBIC_V2_NCW=20" "EBIC_V2_NCW=28" "EBIC_DEBUG_MODE=3" "EBIC_DEBUG_MODE=3 EBIC_V2_NCW=20" "EBIC_DEBUG_MODE=3 EBIC_V2_NCW=28" > gpurun_out/r02_v2f_$w.log 2>&1
done
python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/r02_v2f_bench.log 2>&1
EBIC_PHASE_TIMING=1 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-large > gpurun_out/r02_v2f_phase.log 2>&1
