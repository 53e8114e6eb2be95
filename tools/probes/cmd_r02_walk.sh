mkdir -p gpurun_out
./tools/probes/gather_probe 200000 1000 620 > gpurun_out/r02_gather2.log 2>&1
./tools/probes/gather_probe 20000 500 440 >> gpurun_out/r02_gather2.log 2>&1
for P in 288 576 1152 2048; do python tools/kernel_probe.py synth:200064,500,$P,5 "EBIC_DEBUG_MODE=2" "EBIC_DEBUG_MODE=2 EBIC_SPG=4" >> gpurun_out/r02_walk_scaling.log 2>&1; done
for L in 3 8 12; do python tools/kernel_probe.py synth:200064,500,576,$L "EBIC_DEBUG_MODE=2" >> gpurun_out/r02_walk_scaling.log 2>&1; done
python tools/kernel_probe.py synth:200064,500,576,5 "EBIC_DEBUG_MODE=2 EBIC_NCW=16" "EBIC_DEBUG_MODE=2 EBIC_NCW=32" "" "EBIC_DEBUG_MODE=1" >> gpurun_out/r02_walk_scaling.log 2>&1
