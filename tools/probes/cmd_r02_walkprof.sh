# ncu of the pure walk (EBIC_DEBUG_MODE=2: no loads) on a C4-width synthetic
# matrix with 21 tiles per CTA, so prologue and tail are negligible.
mkdir -p gpurun_out
W="synth:200064,500,576,5"
EBIC_DEBUG_MODE=2 python tools/kernel_probe.py $W > gpurun_out/r02_walkprof_plain.log 2>&1 && \
EBIC_DEBUG_MODE=2 ncu --set full --clock-control none --import-source on -k regex:count_ -s 3 -c 1 -o gpurun_out/prof_r02_walk python tools/kernel_probe.py $W > gpurun_out/ncu_r02_walk.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_r02_walk.log
